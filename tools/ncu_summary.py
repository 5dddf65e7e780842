"""Summarise ncu raw CSV pages (tools/gpu_ncu_set.sh) into one JSON object per capture."""
import csv, json, sys
KEYS = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_pipe_active_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_wavefronts_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__occupancy_limit_shared_mem": "ctas_per_sm_smem_limit",
}
out = {}
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")][:90]}
    for k, name in KEYS.items():
        if k in hdr:
            i = hdr.index(k)
            d[name] = f"{vals[i]} {units[i]}".strip()
    pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
    stalls = {h[len(pre):-len(suf)]: float(vals[i] or 0) for i, h in enumerate(hdr)
              if h.startswith(pre) and h.endswith(suf) and "not_issued" not in h}
    tot = sum(stalls.values()) or 1.0
    d["stall_share_top"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
    out[path.split("/")[-1].replace("_raw.csv", "")] = d
print(json.dumps(out, indent=1))
