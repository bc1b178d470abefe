"""Summarise an .ncu-rep: key metrics per launch, stall reasons, executed SASS by opcode and
the hottest SASS instructions by stall samples.
    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [out_prefix]
"""
import collections, csv, io, re, subprocess, sys

rep = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else None

def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout

raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
hdr, units, rows = raw[0], raw[1], raw[2:]
KEEP = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'launch__registers_per_thread', 'launch__occupancy_limit_registers',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'l1tex__t_sector_hit_rate.pct',
        'lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'lts__d_atomic_input_cycles_active.max.pct_of_peak_sustained_elapsed',
        'lts__t_requests_srcunit_tex_op_red.sum',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum', 'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum',
        'l1tex__lsuin_requests.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed',
        'smsp__inst_executed_op_shared_atom.sum', 'smsp__thread_inst_executed_per_inst_executed.ratio']
KEEP += [h for h in hdr if 'smsp__average_warps_issue_stalled' in h and h.endswith('_per_issue_active.ratio')]
lines = []
lines.append(",".join(["metric", "unit"] + [f"launch{i}" for i in range(len(rows))]))
for k in KEEP:
    if k in hdr:
        i = hdr.index(k)
        lines.append(",".join([k, units[i]] + ['"%s"' % r[i] if ',' in r[i] else r[i] for r in rows]))
text = "\n".join(lines)
print(text)
if out:
    open(out + "_metrics.csv", "w").write(text + "\n")

sass = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "--print-source", "sass"]))))
ks = [i for i, r in enumerate(sass) if r and r[0] == 'Kernel Name']
if ks:
    h = sass[ks[0] + 1]
    seg = sass[ks[0] + 2:(ks[1] if len(ks) > 1 else len(sass))]
    iS, iE, iSm = h.index('Source'), h.index('Instructions Executed'), h.index('# Samples')
    iSt = h.index('Warp Stall Sampling (All Samples)')
    ops, samp = collections.Counter(), collections.Counter()
    tot = 0
    insts = []
    for n, r in enumerate(seg):
        if len(r) <= iE:
            continue
        m = re.match(r'\s*(@!?U?P\d+\s+)?([A-Z0-9_.]+)', r[iS])
        if not m:
            continue
        op = m.group(2).split('.')[0]
        e, s = int(r[iE] or 0), int(r[iSm] or 0)
        ops[op] += e; samp[op] += s; tot += e
        insts.append((s, e, n, r[iS].strip()))
    out_lines = [f"kernel,{sass[ks[0]][1]}", f"static_instructions,{len(insts)}", f"executed_warp_instructions,{tot}",
                 "opcode,executed,share_pct,stall_samples"]
    for op, e in ops.most_common(28):
        out_lines.append(f"{op},{e},{e / tot * 100:.1f},{samp[op]}")
    out_lines.append("top instructions by stall samples: samples,executed,index,sass")
    for s_, e, n, src in sorted(insts, reverse=True)[:40]:
        out_lines.append(f"{s_},{e},{n},\"{src}\"")
    text2 = "\n".join(out_lines)
    print(text2)
    if out:
        open(out + "_sass.csv", "w").write(text2 + "\n")
