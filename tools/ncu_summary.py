"""Summarise an ncu --set full report (first kernel): key throughput metrics + stall reasons.
    python tools/ncu_summary.py gpurun_out/prof_x.ncu-rep [--json out.json --H 8192]"""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct", "launch__grid_size",
        "launch__waves_per_multiprocessor", "smsp__warps_eligible.avg.per_cycle_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def main():
    d = load(sys.argv[1])
    print("kernel:", d.get("Kernel Name", ("?",))[0][:100])
    for k in KEYS:
        if k in d:
            print(f"  {k:70s} {d[k][0]:>16s} {d[k][1]}")
    stalls = []
    for h, (v, u) in d.items():
        if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
            try:
                stalls.append((float(v), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    print("  stalls (warps per issue):", ", ".join(f"{n}={v:.2f}" for v, n in sorted(stalls, reverse=True)[:8]))
    if "--json" in sys.argv:
        H = int(sys.argv[sys.argv.index("--H") + 1]) if "--H" in sys.argv else None
        sites = int(sys.argv[sys.argv.index("--sites") + 1]) if "--sites" in sys.argv else None
        scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1}
        rb = float(d["dram__bytes_read.sum"][0]) * scale[d["dram__bytes_read.sum"][1]]
        wb = float(d["dram__bytes_write.sum"][0]) * scale[d["dram__bytes_write.sum"][1]]
        res = {"report": sys.argv[1], "kernel": d.get("Kernel Name", ("?",))[0], "workload_H": H,
               "dram_bytes_read": rb, "dram_bytes_write": wb, "dram_bytes_per_launch": rb + wb,
               "duration_us_ncu": float(d["gpu__time_duration.sum"][0]),
               "metrics": {k: d[k][0] + " " + d[k][1] for k in KEYS if k in d},
               "stalls": {n: v for v, n in stalls}}
        if sites:
            inst = float(d["smsp__inst_executed.sum"][0])
            res["sites_per_launch"] = sites
            res["thread_instr_per_su"] = 32.0 * inst / sites
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
