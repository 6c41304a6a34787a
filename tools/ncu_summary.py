"""Summarise an .ncu-rep: key metrics + top stall SASS lines.  python tools/ncu_summary.py rep [n_lines]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
        "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct"]
for k in want:
    if k in h:
        i = h.index(k); print(f"{k:90s} {u[i]:>10s} {v[i]}")
st = [(k, v[i]) for i, k in enumerate(h) if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
st = sorted(((float(x.replace(',', '') or 0), k) for k, x in st), reverse=True)[:8]
print("stalls:", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')}={int(c)}" for c, k in st))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = next(r for r in rows if "Address" in r)
ai, si, wi = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[rows.index(hdr) + 1:]:
    try: data.append((int(r[wi]), r[ai], r[si]))
    except Exception: pass
tot = sum(d[0] for d in data) or 1
for d in sorted(data, reverse=True)[:top]: print(f"{d[0]:7d} {100*d[0]/tot:5.1f}% {d[2][:100]}")
