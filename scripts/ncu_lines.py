"""Per source line: executed warp instructions and stall samples of one kernel in an .ncu-rep
(needs -lineinfo).   python scripts/ncu_lines.py rep.ncu-rep [min_share_pct]"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]; thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.8
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = None; hdr = None
agg = collections.OrderedDict()
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": continue
    if r[0] == "Line No": hdr = r; iI = hdr.index("Instructions Executed"); iS = hdr.index("# Samples"); continue
    if r[0] == "" or hdr is None: continue       # sass rows
    try:
        key = (fname, int(r[0]))
    except ValueError:
        continue
    if len(r) != len(hdr):
        continue          # a source line with commas inside quotes that the exporter did not escape
    try:
        e = int(r[iI] or 0); smp = int(r[iS] or 0)
    except ValueError:
        continue
    a = agg.setdefault(key, [0, 0, r[1].strip()[:90]])
    a[0] += e; a[1] += smp
tot = sum(a[0] for a in agg.values()); tots = sum(a[1] for a in agg.values())
print("total executed", tot, "samples", tots)
for (f, ln), (e, smp, src) in agg.items():
    if e / tot * 100 >= thr or smp / max(tots, 1) * 100 >= thr:
        print(f"{f}:{ln:4d} {e/tot*100:5.1f}% inst {smp/max(tots,1)*100:5.1f}% stall  {src}")
