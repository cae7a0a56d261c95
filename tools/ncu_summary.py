"""Summarise an ncu --set full report (one kernel launch) into a small text + json for profiles/."""
import csv, io, json, subprocess, sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__waves_per_multiprocessor",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__warps_active.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    return hdr, units, vals


def main(rep, out_txt, out_json=None, label=""):
    hdr, units, vals = raw(rep)
    res = {}
    with open(out_txt, "w") as f:
        f.write(f"# ncu --set full summary: {rep} {label}\n")
        for v in vals:
            name = v[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
            f.write(f"kernel: {name[:120]}\n")
            for k in KEYS:
                for i, h in enumerate(hdr):
                    if h == k:
                        f.write(f"  {k} = {v[i]} {units[i]}\n")
                        res[k] = v[i]
            stalls = []
            for i, h in enumerate(hdr):
                if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio"):
                    try:
                        stalls.append((float(v[i]), h))
                    except ValueError:
                        pass
            for val, h in sorted(stalls, reverse=True)[:8]:
                f.write(f"  stall {h.replace('smsp__average_warp_latency_issue_stalled_', '')} = {val:.3f}\n")
    if out_json:
        rd = float(res.get("dram__bytes_read.sum", 0) or 0)
        wr = float(res.get("dram__bytes_write.sum", 0) or 0)
        unit = units[hdr.index("dram__bytes_read.sum")]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        json.dump({"report": rep, "label": label, "dram_bytes_per_launch": (rd + wr) * scale,
                   "dram_read_bytes": rd * scale, "dram_write_bytes": wr * scale}, open(out_json, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
