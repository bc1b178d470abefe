"""Static SASS statistics per kernel of libmpm_b200.so: python scripts/sass_stats.py [filter]"""
import collections, re, subprocess, sys
import os
so = os.environ.get("SO", "paper_2111_00699_b200/libmpm_b200.so")
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
flt = sys.argv[1] if len(sys.argv) > 1 else "transfer_kernel"
cur, stats = None, {}
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        stats[cur] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,5}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_]+)", line)
    if m and cur:
        stats[cur][m.group(1)] += 1
for f, c in stats.items():
    if flt in f:
        tot = sum(c.values())
        print(f, "static instr", tot)
        print("   ", ", ".join(f"{k}:{v}" for k, v in c.most_common(24)))
