"""Summarise an .ncu-rep (raw + source pages) into text: `python scripts/ncu_summary.py rep units_per_launch [unit_name]`."""
import csv, io, subprocess, sys
from collections import Counter
rep, units = sys.argv[1], float(sys.argv[2])
uname = sys.argv[3] if len(sys.argv) > 3 else "unit"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, vals = rows[0], rows[2]
keys = ['gpu__time_duration.sum', 'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size',
        'launch__shared_mem_per_block_dynamic', 'launch__shared_mem_per_block_static', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'sm__cycles_elapsed.max',
        'smsp__sass_thread_inst_executed_op_dadd_pred_on.sum', 'smsp__sass_thread_inst_executed_op_dmul_pred_on.sum',
        'smsp__sass_thread_inst_executed_op_dfma_pred_on.sum']
print("kernel:", vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?")
for k in keys:
    if k in hdr:
        i = hdr.index(k)
        print(f"  {k} [{rows[1][i]}] = {vals[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
tot = sum(float(r[ix["Instructions Executed"]] or 0) for r in data)
print(f"  warp instructions executed: {tot:.0f} = {tot / units:.1f} per {uname}")
c, st = Counter(), Counter()
for r in data:
    s = r[ix["Source"]].strip()
    op = (s.split()[1] if s.startswith('@') else s.split()[0]).split('.')[0]
    c[op] += float(r[ix["Instructions Executed"]] or 0)
    st[op] += float(r[ix["# Samples"]] or 0)
for op, v in c.most_common(22):
    print(f"    {op:10s} {v / units:9.1f} per {uname}   stall samples {st[op]:.0f}")
stalls = {h: sum(float(r[ix[h]] or 0) for r in data) for h in hdr if h.startswith("stall_") and "Not" not in h}
print("  stall reasons:", ", ".join(f"{h[6:]}={v:.0f}" for h, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]))
