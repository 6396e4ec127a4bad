"""Summarise an ncu --set full report (.ncu-rep) per kernel launch as JSON lines:
duration, DRAM traffic (read+write, the roofline 'traffic' field), throughput
fractions, occupancy, registers, top stall reasons, tensor-pipe activity."""
import csv, io, json, subprocess, sys

M = {
    "time_us": "gpu__time_duration.sum",
    "dram_read_MB": "dram__bytes_read.sum",
    "dram_write_MB": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "dyn_smem": "launch__shared_mem_per_block_dynamic",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
}
STALL = "smsp__average_warps_issue_stalled_"


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0]}
        for k, col in M.items():
            idx = [i for i, name in enumerate(h) if name == col or name.endswith("." + col)]
            if idx:
                v = r[idx[0]]
                try:
                    d[k] = float(v.replace(",", ""))
                except ValueError:
                    d[k] = v
        st = {c[len(STALL):].replace("_per_issue_active.ratio", ""): float(r[i].replace(",", "") or 0)
              for i, c in enumerate(h) if c.startswith(STALL) and c.endswith("_per_issue_active.ratio")}
        d["top_stalls"] = dict(sorted(st.items(), key=lambda x: -x[1])[:5])
        if "dram_read_MB" in d and "dram_write_MB" in d:
            d["traffic_MB"] = round(d["dram_read_MB"] + d["dram_write_MB"], 3)
        print(json.dumps(d))


if __name__ == "__main__":
    main(sys.argv[1])
