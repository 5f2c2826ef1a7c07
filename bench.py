#!/usr/bin/env python
"""Benchmark of the synchronous lazy-PCA sweep (arXiv 2507.14869) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--sweeps S] [--impl ours|reference]

Metric (BASELINE.json): PCA site-updates per second (SU/s = sites x sweeps / time).

One *step* = one pass of the whole hot path over one batch of
synthetic input: pca_reset (x0 = g, counts = 0, t = 0), S synchronous sweeps with fused MPM
counts, the MPM estimate, and PSNR/SSIM of the LAST and MPM estimates against the truth.

* N = 1: config 3 -- 8192 x 8192 single lattice, l = 2, Moore-8 torus, sigma = 0.5,
  fixed beta = 1.5 (steady-state timing), q = 0.51, MPM counting every sweep.
* N > 1 (torchrun, one process per GPU, NCCL): config 4 weak scaling -- a 32768-wide torus
  of 4096*N rows, row strips of 4096 x 32768 per GPU with a one-row halo exchange per
  sweep over NCCL (P = 8 is exactly 32768^2).

`value` is device-timed (CUDA events on the library's stream, inputs resident in HBM);
`e2e` repeats the step through the same C ABI with pinned HOST buffers (g and truth
host->device, MPM image device->host inside the timed region).  `--impl reference` times
the CPU oracle (oracle/, one core) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PCA site-updates/sec"
UNIT = "site-updates/s"
BYTES_PER_SU = 7  # byte kernel: x_t read (1) + g read (1) + x_{t+1} write (1) + uint16 count RMW (2+2)
# bit-packed kernel (PCA_KERNEL_PACKED, the N = 1 default): x_t, g, x_{t+1} at 1 bit each (3/8) +
# uint8 count-delta RMW (1+1)
BYTES_PER_SU_PACKED = 3 / 8 + 2
KERNEL_BINARY, KERNEL_PACKED = 2, 4


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--sweeps", type=int, default=200, help="PCA sweeps per step")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-variants", action="store_true",
                    help="skip the multi-level variants (C5 per GPU, C3 at l = 5) of the N = 1 line")
    ap.add_argument("--rows-per-thread", type=int, default=0)
    ap.add_argument("--halo", default="nccl", choices=["nccl", "p2p"],
                    help="N > 1: halo rows by NCCL send/recv (default) or stored by the sweep "
                         "kernel straight into the neighbours' memory (pca_attach_peers, CUDA IPC)")
    ap.add_argument("--graphs", type=int, default=None,
                    help="capture each pca_sweep(S) run into a CUDA graph and replay it every step "
                         "(pca_config.graphs); default: on for N = 1, off for row strips (N > 1)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak (default): config 3 at N = 1, config 4's 4096 x 32768 rows per GPU at N > 1; "
                         "strong: the 32768^2 lattice split over the N GPUs (N = 1: on one GPU)")
    ap.add_argument("--variant-only", default=None, choices=["c5", "c3_l5"],
                    help="run ONE run of one multi-level variant and exit (no line): the target "
                         "of the all-launch instruction capture (tools/ncu_variant_summary.py)")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU only (gloo, stub context): exercise the multi-rank orchestration "
                         "(self-launch, strip partition, unique-id broadcast, max-over-ranks "
                         "timing, rank-0 line) without a GPU; the line is marked dry_run")
    return ap.parse_args()


def _free_port() -> int:
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args) -> int | None:
    """`python bench.py --gpus N` outside torchrun (WORLD_SIZE unset) with N > 1: re-launch this
    script as N ranks (one process per GPU) with torch.distributed.run on 127.0.0.1, exactly as
    the driver's torchrun launch would, and pass rank 0's JSON line through.  None when this
    process already is a rank (or N == 1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, cwd=ROOT).returncode


def workload(n_gpus: int, scaling: str = "weak"):
    if scaling == "strong":  # SURVEY 8(d) C4's secondary mode: the 32768^2 lattice fixed
        if 32768 % n_gpus:
            raise SystemExit("--scaling strong splits 32768 rows evenly: N must divide 32768")
        split = (f"row strips {32768 // n_gpus}x32768 per GPU, NCCL halo exchange per sweep"
                 if n_gpus > 1 else "the whole lattice on 1 B200")
        return dict(name=f"config4 strong scaling: 32768x32768 torus, {split}, l=2, Moore-8, sigma=0.5, "
                         f"beta=1.5, q=0.51, MPM every sweep",
                    H=32768, W=32768, rows=32768 // n_gpus, levels=2, nbhd=8, periodic=True, sigma=0.5,
                    beta=1.5, parallelism=f"row-strip x{n_gpus}" if n_gpus > 1 else "1 GPU",
                    scaling="strong")
    if n_gpus == 1:
        return dict(name="config3: 8192x8192 single lattice on 1 B200, l=2, Moore-8 torus, "
                         "sigma=0.5, beta=1.5 fixed, q=0.51, MPM counts every sweep",
                    H=8192, W=8192, rows=8192, levels=2, nbhd=8, periodic=True, sigma=0.5,
                    beta=1.5, parallelism="1 GPU", scaling="weak")
    return dict(name=f"config4 weak scaling: {4096 * n_gpus}x32768 torus (32768 wide), row strips "
                     f"4096x32768 per GPU, NCCL halo exchange per sweep, l=2, Moore-8, sigma=0.5, "
                     f"beta=1.5, q=0.51, MPM every sweep",
                H=4096 * n_gpus, W=32768, rows=4096, levels=2, nbhd=8, periodic=True, sigma=0.5,
                beta=1.5, parallelism=f"row-strip x{n_gpus}", scaling="weak")


def make_inputs(wl, rank):
    import synth

    rows, W = wl["rows"], wl["W"]
    truth = synth.tiled_labels(rows, W, wl["levels"], seed=1000 + rank)
    g = synth.degrade(truth, wl["levels"], wl["sigma"], seed=2000 + rank)
    return truth, g


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"pca_bench_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["stdbuf", "-oL", "nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.fh, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.send_signal(2)
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        self.lines = [ln.strip() for ln in open(self.path)]
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def load_traffic(tag):
    """DRAM bytes per sweep launch of the 8192^2 headline kernel (`tag`: the kernel's name in the
    summary file names) from the committed ncu summaries: preferably a multi-launch capture
    without cache control (the steady state: each launch's dirty lines are written back during
    the next, so writes are counted), else the --set full capture."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"*ncu_full*{tag}*summary*.json"))) + \
        sorted(glob.glob(os.path.join(ROOT, "profiles", f"*dram_multilaunch*{tag}*.json")))
    for f in reversed(files):
        try:
            d = json.load(open(f))
            if d.get("workload_H") == 8192 and d.get("dram_bytes_per_launch"):
                return float(d["dram_bytes_per_launch"]), os.path.relpath(f, ROOT)
        except Exception:
            pass
    return None, None


# Issue peak for ALU-bound kernels: 4 SM sub-partitions per SM, each issuing
# at most one warp instruction per clock (B300_MICROARCH.md "Per-warp issue scheduler"), i.e.
# 148 SMs x 4 x 32 thread-instructions per clock at the max SM clock of MEASURED_PEAKS.json.
def issue_peak():
    try:
        mhz = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"])
    except Exception:
        mhz = 1965.0
    return 148 * 4 * 32 * mhz * 1e6


def load_instr_per_su(tag):
    """thread-instructions per site-update of a variant's sweep kernel from its committed ncu
    summary (profiles/*<tag>*summary*.json: smsp__inst_executed.sum x 32 / sites)."""
    import glob

    pat = f"*ncu_full_{tag}_summary.json" if tag.startswith("sweep_") else f"*ncu_full_variant_{tag}_summary.json"
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", pat)), reverse=True):
        try:
            d = json.load(open(f))
            return float(d["thread_instr_per_su"]), os.path.relpath(f, ROOT)
        except Exception:
            pass
    return None, None


def run_variants(P, torch, dev, stream, only=None, runs=2):
    """The paper's multi-level workloads on one GPU: C5 per GPU (one 512^2 truth,
    l = 5, sigma = 0.25, x 128 noise seeds = 128 chains, Moore-8, free boundary, the paper's
    protocol: 1000 sweeps, beta 1.25 + 0.25 / 250, MPM burn-in 750) and C3 at l = 5 (8192^2
    torus, beta = 1.5, MPM every sweep, 200 sweeps from x0 = g).  Each: device time of one
    timed run (reset + sweeps + fused finalisation) after a warm-up run, SU/s, and the ALU
    roofline of its sweep kernel (instructions per SU from the committed ncu summary x SU/s
    against the issue peak)."""
    import synth

    out = {}
    peak = issue_peak()
    cases = [
        ("c5", "C5 per GPU: 128 chains x 512x512, l=5, sigma=0.25, Moore-8 free, paper protocol "
               "(1000 sweeps, beta 1.25+0.25/250, MPM burn-in 750)", 512, 512, 128, 1000,
         dict(sigma=0.25, mpm_burn_in=750)),
        ("c3_l5", "C3 at l=5: 8192x8192 torus, sigma=0.25, beta=1.5, MPM every sweep, 200 sweeps "
                  "from x0 = g", 8192, 8192, 1, 200,
         dict(sigma=0.25, periodic=True, beta0=1.5, beta_step=0.0, mpm_burn_in=0)),
    ]
    for tag, name, H, W, B, S, kw in cases:
        if only is not None and tag != only:
            continue
        if B > 1:
            truth1 = synth.smooth_labels(H, W, 5, seed=7)
            truth = np.repeat(truth1[None], B, 0)
            g = np.stack([synth.degrade(truth1, 5, 0.25, seed=100 + b) for b in range(B)])
        else:
            truth = synth.tiled_labels(H, W, 5, seed=1)[None]
            g = synth.degrade(truth[0], 5, 0.25, seed=2)[None]
        gd = torch.from_numpy(np.ascontiguousarray(g)).to(dev)
        td = torch.from_numpy(np.ascontiguousarray(truth)).to(dev)
        mpm = torch.empty_like(gd)
        ctx = P.PcaContext(P.make_config(H, W, 5, batch=B, seed=11, **kw), gd, stream=stream)
        ms = []
        for _ in range(runs):
            ctx.pca_reset(None, None)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ctx.pca_sweep(S)
            psnr, ssim = ctx.pca_finalize(td, mpm)
            b.record(stream)
            torch.cuda.synchronize(dev)
            ms.append(a.elapsed_time(b))
        su_s = B * H * W * S / (ms[-1] * 1e-3)
        ipsu, src = load_instr_per_su(tag)
        roof = None
        if ipsu:
            roof = {"bound": "alu", "achieved": ipsu * su_s, "peak": peak, "unit": "thread-instr/s",
                    "frac": ipsu * su_s / peak, "instr_per_su": ipsu, "instr_source": src,
                    "peak_source": "148 SMs x 4 schedulers x 32 lanes x sm_max_mhz (1 warp-instr/clk/SMSP)"}
        out[tag] = {"workload": name, "value": su_s, "unit": UNIT, "ms_per_run": ms[-1],
                    "us_per_sweep": 1e3 * ms[-1] / S, "sweeps": S,
                    "psnr_ssim_mpm_chain0": [float(psnr[0, 1]), float(ssim[0, 1])],
                    "roofline": roof}
        ctx.pca_destroy()
        del gd, td, mpm
    return out


def measured_peak():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---------------------------------------------------------------------------
def host_cpu():
    """The host CPU model and the number of online cores (nproc)."""
    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model, os.cpu_count()


def cpu_baseline_oracle(wl, truth, g, rows=None, sweeps=2):
    """The oracle, as it stands (single-threaded C, fp64), on a bounded sample of the
    workload: `sweeps` sweeps of the first `rows` rows treated as their own torus.  The
    process is pinned to ONE core (sched_setaffinity) for the timed call."""
    import oracle as orc

    rows = rows or wl["rows"]
    m = orc.model(rows, wl["W"], wl["levels"], nbhd=wl["nbhd"], periodic=wl["periodic"],
                  sigma=wl["sigma"], q=0.51)
    gs = np.ascontiguousarray(g[:rows])
    ts = np.ascontiguousarray(truth[:rows])
    old = os.sched_getaffinity(0)
    core = min(old)
    os.sched_setaffinity(0, {core})
    try:
        t0 = time.perf_counter()
        x, cnt = orc.pca_run(m, gs, gs, sweeps, wl["beta"], 0.0, 1 << 30, 11, burn_in=0)
        orc.metrics(ts, x, wl["levels"])                # LAST
        orc.metrics(ts, orc.mpm(cnt), wl["levels"])     # MPM (argmax of the counts)
        dt = time.perf_counter() - t0
    finally:
        os.sched_setaffinity(0, old)
    su = rows * wl["W"] * sweeps
    model, nproc = host_cpu()
    return {"value": su / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "cpu_model": model, "nproc": nproc, "pinned_core": core,
            "sample": f"{sweeps} oracle sweeps (+MPM counts, MPM image, metrics of LAST and MPM) of a {rows}x{wl['W']} "
                      f"torus cut from the same input, 1 thread pinned to core {core} of {nproc} "
                      f"({model}), {dt:.1f} s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    wl = workload(args.gpus, args.scaling)
    truth, g = make_inputs(wl, 0)
    rows = 512
    times = []
    for i in range(args.warmup + args.steps):
        r = cpu_baseline_oracle(wl, truth, g, rows=rows, sweeps=1)
        if i >= args.warmup:
            times.append(r)
    vals = [r["value"] for r in times]
    v = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * rows * wl["W"] / v,
        "higher_is_better": True, "scaling": wl["scaling"], "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": wl["name"], "H": wl["H"], "W": wl["W"],
                                        "reference_sample_rows": rows, "sweeps_per_step": 1},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "cpu_model": times[0]["cpu_model"], "nproc": times[0]["nproc"],
                         "sample": f"each step: 1 oracle sweep (+MPM, +metrics) of a {rows}x"
                                   f"{wl['W']} torus cut from the workload, 1 thread pinned to "
                                   f"one core"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
def run_ours(args):
    import torch

    import paper_2507_14869_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n = max(args.gpus, world)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        # the strips' halo send/recv kernels must fit beside the resident interior sweep (one
        # wave of 14 one-warp CTAs per SM leaves ~17 K registers per SM): small NCCL blocks
        #
        os.environ.setdefault("NCCL_NTHREADS", "128")
        dist.init_process_group("nccl", device_id=dev)
    from paper_2507_14869_b200 import dist as pdist

    wl = workload(n, args.scaling)
    truth, g = make_inputs(wl, rank)
    rows, W = wl["rows"], wl["W"]
    assert pdist.strip_rows(wl["H"], max(world, 1), rank)[1] == rows
    stream = torch.cuda.Stream(device=dev)
    g_dev = torch.from_numpy(g).to(dev).reshape(1, rows, W).contiguous()
    t_dev = torch.from_numpy(truth).to(dev).reshape(1, rows, W).contiguous()
    mpm_dev = torch.empty_like(g_dev)
    graphs = args.graphs if args.graphs is not None else (1 if world == 1 else 0)
    kw = dict(neighborhood=wl["nbhd"], periodic=wl["periodic"], sigma=wl["sigma"], q=0.51,
              beta0=wl["beta"], beta_step=0.0, beta_period=1 << 30, seed=11, mpm_burn_in=0,
              rows_per_thread=args.rows_per_thread, graphs=graphs if wl["levels"] == 2 else 0)
    peers = []
    if world > 1:  # this rank's row strip, NCCL attached (unique id broadcast by torch.distributed)
        ctx = pdist.strip_context(kw, wl["H"], W, wl["levels"], g_dev, stream=stream)
        if args.halo == "p2p":  # halo rows stored by the sweep kernels into the neighbours' memory
            peers += pdist.attach_peers_ipc(ctx, kw, wl["H"], W, wl["levels"])
    else:
        ctx = P.PcaContext(P.make_config(wl["H"], W, wl["levels"], **kw), g_dev, stream=stream)
    S = args.sweeps

    def step_device():
        ctx.pca_reset(None, None)
        ctx.pca_sweep(S)
        return ctx.pca_finalize(t_dev, mpm_dev)  # MPM image + PSNR/SSIM of LAST and MPM

    def barrier():
        torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(v):
        if not dist:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-timed run ----
    for _ in range(args.warmup):
        step_device()
    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    st0 = ctx.pca_get_stats()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sw_ms = 0.0
    ev0.record(stream)
    for _ in range(args.steps):
        ctx.pca_reset(None, None)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ctx.pca_sweep(S)
        b.record(stream)
        psnr, ssim = ctx.pca_finalize(t_dev, mpm_dev)  # synchronises the stream
        sw_ms += a.elapsed_time(b)
    ev1.record(stream)
    barrier()
    st1 = ctx.pca_get_stats()
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    sw_ms = max_over_ranks(sw_ms)
    sites_all = wl["H"] * W
    value = sites_all * S * args.steps / (ms * 1e-3)
    launches = int(st1.kernel_launches - st0.kernel_launches)

    # roofline of the dominant kernel (the fused sweep).  sweep_s = the mean time per sweep of
    # the pca_sweep(S) calls (CUDA events on the library's stream; for the packed kernel it
    # includes the pack / unpack / count-fold passes of each call)
    sweep_s = sw_ms * 1e-3 / (S * args.steps)
    kernel_used = int(st1.kernel)
    packed_k = kernel_used == KERNEL_PACKED
    bpsu = BYTES_PER_SU_PACKED if packed_k else BYTES_PER_SU
    tag = "sweep_packed" if packed_k else "sweep_binary"
    alg_bytes = bpsu * rows * W
    peak, peak_src = measured_peak()
    achieved = alg_bytes / sweep_s / 1e9
    traffic, traffic_src = load_traffic(tag)
    hbm_roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "frac_dram": (traffic / sweep_s / 1e9 / peak) if traffic else None,
                "bytes_per_launch_alg": alg_bytes, "alg_bytes_per_site_update": bpsu,
                "mean_launch_us": sweep_s * 1e6, "peak_source": peak_src,
                "traffic_source": traffic_src}
    if packed_k:
        # the packed kernel moves 2.375 B/SU and is bound by instruction issue: its roofline is
        # thread-instructions per SU (committed ncu summary) x SU/s against the issue peak
        ipsu, isrc = load_instr_per_su(tag)
        ipk = issue_peak()
        roofline = {"bound": "alu", "kernel": "sweep_packed_kernel (bit-packed PCA sweep + uint8 MPM "
                                              "count deltas)",
                    "achieved": (ipsu * rows * W / sweep_s) if ipsu else None, "peak": ipk,
                    "unit": "thread-instr/s", "frac": (ipsu * rows * W / sweep_s / ipk) if ipsu else None,
                    "traffic": traffic, "instr_per_su": ipsu, "instr_source": isrc,
                    "mean_launch_us": sweep_s * 1e6,
                    "peak_source": "148 SMs x 4 schedulers x 32 lanes x sm_max_mhz (1 warp-instr/clk/SMSP)",
                    "hbm": hbm_roof}
    else:
        roofline = dict(hbm_roof, kernel="sweep_binary_kernel (fused PCA sweep + MPM counts)")

    # ---- end-to-end through the C ABI with pinned host buffers.  Two-level images travel
    # bit-packed (pca_config.packed_io): 1 bit per site in each direction ----
    e2e = None
    if not args.no_e2e:
        packed = wl["levels"] == 2
        kw_e = dict(kw, packed_io=int(packed))
        pk = P.pack_bits if packed else (lambda a: a)
        g_h = torch.from_numpy(np.ascontiguousarray(pk(g))).reshape(1, rows, -1).pin_memory()
        t_h = torch.from_numpy(np.ascontiguousarray(pk(truth))).reshape(1, rows, -1).pin_memory()
        mpm_h = torch.empty(tuple(t_h.shape), dtype=torch.uint8).pin_memory()
        if world > 1:
            ectx = pdist.strip_context(kw_e, wl["H"], W, wl["levels"], g_h, stream=stream)
            if args.halo == "p2p":
                peers += pdist.attach_peers_ipc(ectx, kw_e, wl["H"], W, wl["levels"])
        else:
            ectx = P.PcaContext(P.make_config(wl["H"], W, wl["levels"], **kw_e), g_h, stream=stream)

        def step_e2e():
            ectx.pca_reset_staged()              # this step's g (its H2D ran during the last step)
            ectx.pca_stage_input(g_h)            # H2D of the next step's g, overlapping the sweeps
            ectx.pca_stage_truth(t_h)            # H2D of the truth, overlapping the sweeps
            ectx.pca_sweep(S)
            # D2H of the MPM image on the copy stream, overlapping the next step's sweeps
            return ectx.pca_finalize_async(None, mpm_h)

        ectx.pca_stage_input(g_h)                # the first step's input

        for _ in range(max(1, args.warmup)):
            step_e2e()
        ectx.pca_sync()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            pe, se = step_e2e()
        ectx.pca_sync()                          # the last step's MPM image is on the host
        e1.record(stream)
        barrier()
        ems = max_over_ranks(e0.elapsed_time(e1))
        assert abs(pe[0, 1] - psnr[0, 1]) < 1e-9 and abs(se[0, 1] - ssim[0, 1]) < 1e-12  # same chain
        # the MPM image that came back asynchronously is the device-timed run's
        assert np.array_equal(mpm_h.numpy().reshape(-1),
                              np.asarray(pk(mpm_dev.cpu().numpy())).reshape(-1)), "e2e MPM image differs"
        e2e = {"value": sites_all * S * args.steps / (ems * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(g_h.numel() + t_h.numel()),
               "d2h_bytes_per_step": int(mpm_h.numel() + 4 * 8),
               "ms_per_step": ems / args.steps,
               "io": ("bit-packed images (packed_io): g and truth in, MPM image out, 1 bit per site"
                      if packed else "dense uint8 images") +
                     "; each step copies the next step's g and its own truth on a copy stream "
                     "overlapping its sweeps (pca_stage_input / pca_stage_truth); its MPM image "
                     "comes back on the copy stream during the next step (pca_finalize_async), "
                     "the last one inside the timed region (pca_sync before the end event)"}
        ectx.pca_destroy()

    clk = clocks.stop()

    # ---- exposed halo exchange (N > 1): the same strip swept as an isolated torus of
    # rows x W (identical kernels, no NCCL) vs the sharded sweeps timed above ----
    halo = None
    if world > 1:
        local = P.PcaContext(P.make_config(rows, W, wl["levels"], **kw), g_dev, stream=stream)
        local.pca_sweep(S)
        barrier()
        l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0.record(stream)
        for _ in range(args.steps):
            local.pca_sweep(S)
        l1.record(stream)
        barrier()
        local_us = max_over_ranks(l0.elapsed_time(l1)) * 1e3 / (S * args.steps)
        local.pca_destroy()
        halo = {"sweep_us_sharded": sweep_s * 1e6, "sweep_us_local_only": local_us,
                "exposed_us_per_sweep": sweep_s * 1e6 - local_us,
                "messages_per_sweep_per_rank": 4, "bytes_per_message": 16 * ((W + 15) // 16) + 32,  # one padded row (depth 1)
                "halo_exchange": args.halo,
                "method": ("max over ranks of S sharded sweeps (edge rows + NCCL send/recv "
                           "overlapping the interior)" if args.halo == "nccl" else
                           "max over ranks of S sharded sweeps (one launch per sweep storing the "
                           "edge rows into the neighbours' halo rows over peer memory, stream "
                           "waits/writes of phase words)") +
                          " minus S sweeps of the same strip as an isolated torus (no exchange)"}

    variants = None
    if rank == 0 and n == 1 and not args.no_variants:
        variants = run_variants(P, torch, dev, stream)
        if packed_k:
            # the same sweeps on the byte-state kernel (round 1's headline, HBM-bound at 7 B/SU):
            # its time and HBM fraction, for continuity with the packed kernel's issue roofline
            bctx = P.PcaContext(P.make_config(wl["H"], W, wl["levels"], **dict(kw, kernel=KERNEL_BINARY,
                                                                               graphs=0)), g_dev, stream=stream)
            bctx.pca_sweep(10)
            bctx.pca_reset(None, None)
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            b0.record(stream)
            bctx.pca_sweep(S)
            b1.record(stream)
            torch.cuda.synchronize(dev)
            bs = b0.elapsed_time(b1) * 1e-3 / S
            bt, bsrc = load_traffic("sweep_binary")
            variants["byte_state_kernel"] = {
                "workload": wl["name"] + " (the byte-state kernel, PCA_KERNEL_BINARY)",
                "us_per_sweep": bs * 1e6, "value": rows * W / bs, "unit": UNIT,
                "roofline": {"bound": "hbm", "achieved": BYTES_PER_SU * rows * W / bs / 1e9, "peak": peak,
                             "unit": "GB/s", "frac": BYTES_PER_SU * rows * W / bs / 1e9 / peak,
                             "alg_bytes_per_site_update": BYTES_PER_SU, "traffic": bt, "traffic_source": bsrc}}
            bctx.pca_destroy()

    cpu = None
    if rank == 0 and n == 1 and not args.no_cpu_baseline:
        # ~14 s of CPU work: 3 sweeps of at most 2^26 sites (8192^2; 2048 rows at 32768 wide)
        cpu = cpu_baseline_oracle(wl, truth, g, rows=min(wl["rows"], (1 << 26) // wl["W"]), sweeps=3)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": wl["scaling"], "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": wl["name"], "H": wl["H"], "W": W, "rows_per_gpu": rows,
                       "levels": wl["levels"], "sweeps_per_step": S,
                       "step": "reset + S fused sweeps (MPM on) + fused finalisation (MPM image, "
                               "PSNR/SSIM of LAST and MPM in one pass)",
                       "l2": ("no flush: every step starts by rewriting the byte state and the counts "
                              "(192 MiB > 126 MB L2) and ends with the finalisation pass (~320 MiB); "
                              "inside a step the packed kernel's per-sweep working set (2 x 8.4 MiB "
                              "packed state, 8 MiB packed g, 64 MiB count deltas) is L2-sized, which "
                              "is the method's own reuse" if packed_k else
                              "working set ~320 MiB/GPU > 126 MB L2: inputs larger than L2, no flush"),
                       "kernel": {KERNEL_PACKED: "PACKED", KERNEL_BINARY: "BINARY"}.get(kernel_used, kernel_used),
                       "cuda_graphs": bool(kw["graphs"]),
                       "graph_replays": int(st1.graph_replays - st0.graph_replays),
                       "parallelism": wl["parallelism"] + (f", halo {args.halo}" if world > 1 else ""),
                       "psnr_ssim_last": [float(psnr[0, 0]), float(ssim[0, 0])],
                       "psnr_ssim_mpm": [float(psnr[0, 1]), float(ssim[0, 1])]},
            "roofline": roofline,
            "gpu_launches": launches,
            "e2e": e2e,
            "halo": halo,
            "clocks": clk,
            "cpu_baseline": cpu,
            "variants": variants,
        }
        print(json.dumps(line), flush=True)
    ctx.pca_destroy()
    if dist:
        dist.barrier()  # every rank's stores into its neighbours' memory are complete
        for q in peers:
            P.pca_close_peer(q)
        dist.destroy_process_group()
    return 0


def run_dry(args):
    """--dry-run: the multi-rank orchestration of run_ours on CPU (gloo), with a stub in place
    of the CUDA context: ranks from the launcher's environment, the workload for N ranks, this
    rank's strip from dist.strip_rows, the NCCL unique id broadcast (created through the C ABI,
    which needs no GPU), timed stub steps, max over ranks, one line from rank 0."""
    import torch
    import torch.distributed as dist

    from paper_2507_14869_b200 import dist as pdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    n = max(args.gpus, world)
    if world > 1:
        dist.init_process_group("gloo")
    wl = workload(n, args.scaling)
    row0, rows = pdist.strip_rows(wl["H"], world, rank)
    assert rows == wl["rows"], (rows, wl["rows"])
    uid = pdist.broadcast_unique_id() if world > 1 else b""
    up, down = pdist.ring_peers(rank, world, wl["periodic"])

    class StubStrip:  # what the step calls on a PcaContext, without device work
        def __init__(self):
            self.sweeps = 0

        def pca_reset(self, g=None, x0=None):
            self.sweeps = 0

        def pca_sweep(self, k):
            self.sweeps += k

        def pca_finalize(self, truth, out):
            return np.zeros((1, 2)), np.zeros((1, 2))

    ctx = StubStrip()
    t0 = time.perf_counter()
    for _ in range(args.warmup + args.steps):
        ctx.pca_reset()
        ctx.pca_sweep(args.sweeps)
        ctx.pca_finalize(None, None)
    ms = 1e3 * (time.perf_counter() - t0)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        got = [None] * world
        dist.all_gather_object(got, (rank, row0, rows, up, down, len(uid)))
    else:
        got = [(0, row0, rows, up, down, 0)]
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "value": None, "unit": UNIT,
                          "n_gpus": n, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": ms / max(1, args.warmup + args.steps), "scaling": wl["scaling"],
                          "config": {"workload": wl["name"], "H": wl["H"], "W": wl["W"],
                                     "rows_per_gpu": rows, "parallelism": wl["parallelism"]},
                          "ranks": [{"rank": r, "row0": a, "rows": b, "up": u, "down": d,
                                     "unique_id_bytes": k} for r, a, b, u, d, k in got],
                          "stub_sweeps_per_step": ctx.sweeps}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    rc = self_launch(args)
    if rc is not None:
        return rc
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.variant_only:
        import torch

        import paper_2507_14869_b200 as P

        dev = torch.device("cuda", 0)
        stream = torch.cuda.Stream(device=dev)
        out = run_variants(P, torch, dev, stream, only=args.variant_only, runs=1)
        print(json.dumps({k: {"us_per_sweep": v["us_per_sweep"], "sweeps": v["sweeps"]} for k, v in out.items()}))
        return 0
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
