#!/bin/bash
# two ranks sharing ONE GPU (functional stand-in for two GPUs): frame time of the peer-mapped path.
# The contexts are time-sliced, so only the HOST side of the collective steps shows up here.
MPM_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port ${1:-29710} bench.py --gpus 2 --steps 6 --warmup 3 --no-e2e 2>&1 | \
  grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('2 ranks / 1 GPU: frame %.2f ms, value %.0f, rebuilds %s' % (d['ms_per_step'], d['value'], d['config'].get('rebuilds_in_timed_region')))"
