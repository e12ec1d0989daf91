"""Summarise an ncu report: key throughput metrics, stall reasons, top stalled SASS, instruction mix."""
import csv, subprocess, sys
from collections import Counter

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return [dict(zip(r[0], row)) for row in r[2:]]

def num(v):
    try: return float(v.replace(',', ''))
    except Exception: return None

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg.per_second", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]

def main(rep, kernel_filter=None):
    for d in raw(rep):
        name = d.get("Kernel Name", "")
        if kernel_filter and kernel_filter not in name: continue
        print("==", name[:100])
        for k in KEYS:
            if k in d: print(f"  {k:75s} {d[k]}")
        st = [(num(v), k) for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and num(v)]
        tot = sum(v for v, _ in st)
        print("  stalls:", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_','')} {v/tot*100:.1f}%" for v, k in sorted(st, reverse=True)[:8]))
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3: return
    hdr = rows[1]; data = rows[2:]
    i_src, i_s, i_ex = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    tot = sum(num(r[i_s]) or 0 for r in data)
    print("  top stalled SASS:")
    for r in sorted(data, key=lambda r: -(num(r[i_s]) or 0))[:12]:
        print(f"    {(num(r[i_s]) or 0)/tot*100:5.1f}%  {r[i_src][:100]}")
    c = Counter()
    for r in data:
        toks = r[i_src].split()
        if not toks: continue
        op = toks[1] if toks[0].startswith('@') else toks[0]
        c[op.split('.')[0]] += num(r[i_ex]) or 0
    t = sum(c.values())
    print("  inst mix:", ", ".join(f"{k} {v/t*100:.1f}%" for k, v in c.most_common(12)))

if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
