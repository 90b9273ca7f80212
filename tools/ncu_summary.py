"""Summarise ncu --set full reports (one row per launch) -> JSON (development + profiles/)."""
import csv, io, json, subprocess, sys
KEYS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_bytes": ("dram__bytes_read.sum", 1),
    "dram_write_bytes": ("dram__bytes_write.sum", 1),
    "dram_pct_peak": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "tensor_pipe_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "issue_active_pct": ("sm__inst_issued.avg.pct_of_peak_sustained_active", 1),
    "l1_smem_pct": ("l1tex__throughput.avg.pct_of_peak_sustained_active", 1),
    "lts_hit_pct": ("lts__t_sector_hit_rate.pct", 1),
    "registers": ("launch__registers_per_thread", 1),
    "grid": ("launch__grid_size", 1),
    "cluster": ("launch__cluster_dim_x", 1),
    "smem_bytes": ("launch__shared_mem_per_block_dynamic", 1),
}
def unit_scale(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Kbyte/block": 1e3,
            "us": 1e3, "ms": 1e6, "ns": 1, "usecond": 1e3, "msecond": 1e6, "nsecond": 1,
            "%": 1, "": 1}.get(u, 1)
def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": r[hdr.index("Kernel Name")][:60]}
        for k, (m, _) in KEYS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", "")) * unit_scale(units[i])
                except ValueError:
                    continue
                if k == "duration_us":
                    v = v / 1e3  # ns -> us
                d[k] = v
        stalls = {h.split("smsp__average_warps_issue_stalled_")[1].split("_per")[0]: float(r[i] or 0)
                  for i, h in enumerate(hdr)
                  if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")}
        d["top_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda x: -x[1])[:5])
        res.append(d)
    return res
if __name__ == "__main__":
    out = {rep: load(rep) for rep in sys.argv[1:]}
    print(json.dumps(out, indent=1))
