"""Instructions per site-update of a multi-level variant over EVERY sweep launch of one run
(the all-launch capture), for bench.py's variant rooflines (developer tool):

    ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none \\
        -k regex:sweep_ --csv --log-file gpurun_out/var_c5.csv \\
        python bench.py --variant-only c5
    python tools/ncu_variant_summary.py gpurun_out/var_c5.csv c5 profiles/r02_ncu_full_variant_c5_summary.json

thread_instr_per_su = 32 x sum(smsp__inst_executed.sum) / (sites x sweeps), i.e. the mean over
the whole protocol (noisy first sweeps, every beta stage, counting and non-counting sweeps)
rather than one sampled launch.  The ncu durations are serialised and cold-cache, so only
their shares are reported."""
import csv
import json
import sys
from collections import defaultdict

# (sites per sweep, sweeps per run) of bench.py's variants
SHAPES = {"c5": (128 * 512 * 512, 1000), "c3_l5": (8192 * 8192, 200)}


def main():
    path, tag, out = sys.argv[1], sys.argv[2], sys.argv[3]
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    hdr = rows[0]
    ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    inst, dur, count = defaultdict(float), defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        name = r[ik].split("(")[0].replace("void ", "")
        v = float(r[iv].replace(",", ""))
        if r[im] == "smsp__inst_executed.sum":
            inst[name] += v
            count[name] += 1
        elif r[im] == "gpu__time_duration.sum":
            dur[name] += v
    sites, sweeps = SHAPES[tag]
    tot = sum(inst.values())
    launches = sum(count.values())
    res = {"source": path, "workload": tag, "sites_per_sweep": sites, "sweeps": sweeps,
           "sweep_launches": launches, "thread_instr_per_su": 32.0 * tot / (sites * sweeps),
           "method": "32 x sum of smsp__inst_executed.sum over every sweep-kernel launch of one "
                     "run / (sites x sweeps)",
           "kernels": {k: {"launches": count[k], "warp_instructions": inst[k],
                           "share_of_instructions": inst[k] / tot,
                           "share_of_ncu_time": dur[k] / max(sum(dur.values()), 1e-30)}
                       for k in sorted(inst)}}
    if launches != sweeps:
        res["note"] = f"{launches} sweep launches for {sweeps} sweeps"
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({k: res[k] for k in ("sweep_launches", "thread_instr_per_su")}))


if __name__ == "__main__":
    main()
