"""Per-launch DRAM traffic of consecutive sweep launches captured WITHOUT cache control
(ncu --cache-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,
gpu__time_duration.sum -k regex:<kernel> -c N --csv): the steady state, in which each launch's
dirty lines are written back during the next launches, so writes are counted (a single flushed
capture leaves them in L2).  Launches after the first are averaged.

    python tools/ncu_dram_multi.py launches.csv --out profiles/x.json --H 8192 --sites N
"""
import csv
import json
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
         "msecond": 1e3}


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    per = {}
    for r in rows[1:]:
        lid = int(r[ix["ID"]])
        per.setdefault(lid, {"kernel": r[ix["Kernel Name"]]})[r[ix["Metric Name"]]] = \
            float(r[ix["Metric Value"]].replace(",", "")) * SCALE.get(r[ix["Metric Unit"]], 1.0)
    launches = [per[k] for k in sorted(per)]
    steady = launches[1:] if len(launches) > 1 else launches
    rd = sum(l["dram__bytes_read.sum"] for l in steady) / len(steady)
    wr = sum(l["dram__bytes_write.sum"] for l in steady) / len(steady)
    us = sum(l["gpu__time_duration.sum"] for l in steady) / len(steady)
    out = {"source": sys.argv[1], "kernel": launches[0]["kernel"], "launches": len(launches),
           "averaged_launches": len(steady), "dram_bytes_read": rd, "dram_bytes_write": wr,
           "dram_bytes_per_launch": rd + wr, "duration_us_ncu": us,
           "dram_GBps_at_ncu_time": (rd + wr) / us / 1e3,
           "note": "ncu --cache-control none: consecutive launches, L2 not flushed"}
    if "--H" in sys.argv:
        out["workload_H"] = int(sys.argv[sys.argv.index("--H") + 1])
    if "--sites" in sys.argv:
        n = int(sys.argv[sys.argv.index("--sites") + 1])
        out["dram_bytes_per_su"] = (rd + wr) / n
    print(json.dumps(out, indent=1))
    if "--out" in sys.argv:
        json.dump(out, open(sys.argv[sys.argv.index("--out") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
