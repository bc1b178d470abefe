#!/bin/bash
# build a kernel-experiment variant of the library: scripts/build_variant.sh <name> [-DMPM_TW=4 ...]
# -> paper_2111_00699_b200/variants/libmpm_<name>.so (select with MPM_B200_LIB=...)
name=$1; shift
cd "$(dirname "$0")/../paper_2111_00699_b200" && mkdir -p variants
python - "$name" "$@" <<'PY'
import sys, os
sys.path.insert(0, os.path.dirname(os.getcwd()))
from paper_2111_00699_b200 import build as B
name, extra = sys.argv[1], sys.argv[2:]
B.OUT = os.path.join(B.HERE, "variants", "libmpm_%s.so" % name)
B.OBJ_DIR = os.path.join(B.HERE, "build", "variant_" + name)
import io, contextlib
err = io.StringIO()
old = sys.stderr; sys.stderr = err
try:
    B.build(force=True, verbose=True, extra=extra)
finally:
    sys.stderr = old
open(os.path.join(B.HERE, "variants", name + ".ptxas.log"), "w").write(err.getvalue())
PY
grep -A1 "transfer_kernelILi[12]ELb1ELb1ELb0" variants/$name.ptxas.log | grep -E "spill" | sed "s/^/$name: /"
grep -A2 "transfer_kernelILi[12]ELb1ELb1ELb0" variants/$name.ptxas.log | grep -E "Used" | sed "s/^/$name: /"
