#!/usr/bin/env python
"""Benchmark: Hessian-column applies/s (and member-PCG solves/s) of one
ensemble data-assimilation pass on BASELINE.json config 4 ("Throughput
config": Lorenz-96 n=16384, 24-step window, every 4th variable at every 3rd
step, Gaussian B L=16, 200 members with their own trajectories, rank-128
LMP from a 128-column rhs-difference sketch, 80 PCG iterations batched over
all members, fp64).

One step = one full pass (engine.EdaPass.run):
    rhs of control + all members (one batched AD launch)
    -> Gamma -> Y = A_control Gamma, Nystrom EVD, halfsum LMP
    -> batched LMP-PCG for every member, J traced at every iteration.
value = (ell + members * iters) Hessian-column applies / step time (whole
job, timed as the max over ranks).  ``per_config`` repeats the measurement
for the other BASELINE configs (cfg5: the HBM-scale one) in the same
process.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--scaling weak|strong] [--per-config 1,2,3,5]

--impl reference times the UNMODIFIED reference (edasketch, installed into
baseline/_ref by pip) on the box's host cores for the same metric/config --
its own MemberProblem.hessian_apply / quadratic_cost and krylov.pcg with a
SpectralLmp, one member per process -- rank 0 only; if baseline/_ref is
missing it falls back to the oracle port (kind "port").
"Measurement".
"""

import argparse
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Hessian-column applies/sec and member-PCG solves/sec; % of fp64/HBM roofline"
UNIT = "Hessian-column applies/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--kernel-reps", type=int, default=10)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: cfg.members per GPU; strong: cfg.members sharded over the GPUs")
    ap.add_argument("--per-config", default="1,2,3,5",
                    help="other BASELINE configs measured in the same process ('' = none)")
    return ap.parse_args()


def config_dict(cfg, world, scaling="weak"):
    total = cfg.members * world if scaling == "weak" else cfg.members
    per_gpu = total / world
    traj_gb = (per_gpu + 1) * (cfg.n_steps + 1) * cfg.n * 8 / 1e9
    return {
        "workload": f"BASELINE.json configs[{cfg.name[-1]}-1] ({cfg.name}): Lorenz-96 4D-Var EDA, "
                    "one pass = rhs + Nystrom LMP + batched LMP-PCG",
        "n": cfg.n, "window_steps": cfg.n_steps, "obs_every_var": cfg.obs_stride,
        "obs_every_step": cfg.obs_every, "gaussian_L": cfg.cov_length,
        "members": total, "members_per_gpu": per_gpu,
        "trajectories": "shared control" if cfg.shared_linearization else "per-member",
        "sketch_ell": cfg.ell, "lmp_rank": cfg.k,
        "pcg_iters": cfg.pcg_iters, "theta_rule": "halfsum", "cost_trace": True,
        "parallelism": (f"members sharded over {world} GPUs ({scaling} scaling)" if world > 1
                        else "1 GPU"),
        "l2_policy": (f"inputs larger than L2 (member trajectories {traj_gb:.2f} GB/GPU streamed "
                      "every PCG iteration)" if traj_gb > 0.126 else
                      f"working set {traj_gb * 1e3:.1f} MB/GPU fits in L2 (126 MB): "
                      "L2-resident by construction, like the reference's cache-resident CPU run"),
    }


# ---------------------------------------------------------------- clocks --
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region.

    nvidia-smi needs a few hundred ms to print its first line, which is most
    of a default 5-step timed region, so the sampler is started before the
    warm-up passes (the same load) and every line is stamped on arrival;
    stop(t0, t1) keeps the samples that arrived inside the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def stop(self, t0=None, t1=None):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = list(self.lines)
        window = "timed region"
        if t0 is not None:
            # a line printed at t describes the ~50 ms before it
            inside = [(t, ln) for t, ln in lines if t0 <= t <= t1 + 0.05]
            if inside:
                lines = inside
            else:
                window = "warm-up + timed region (no line arrived inside the timed region)"
        for _, ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "window": window}


# ------------------------------------------------------------ CPU legs ----
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_available():
    """The unmodified reference package, pip-installed into baseline/_ref
    (git-ignored; it travels to the GPU box with the repo snapshot)."""
    return os.path.isfile(os.path.join(REF_DIR, "edasketch", "krylov.py"))


def _gaussian_symbol(n, sigma_b, length):
    """sigma_b sqrt(c_hat): the closed-form (Poisson-summed) DFT of the
    periodic Gaussian correlation row (the same
    adapter tests/golden/make_golden.py gives the reference)."""
    m = np.arange(n // 2 + 1, dtype=float) / n
    c = np.zeros_like(m)
    for k in range(-3, 4):
        c += np.exp(-2.0 * np.pi ** 2 * length ** 2 * (m - k) ** 2)
    return sigma_b * np.sqrt(np.sqrt(2.0 * np.pi) * length * c)


def _ref_member(cfg, j, truth):
    """Member j of a BASELINE config built with the REFERENCE's own
    functions (eda.py:87-108 streams; model.integrate; ObsNetwork;
    MemberProblem), with the Gaussian-symbol adapter on its GridCovFactor
    (the factor duck type covariance.py:41-45 reads)."""
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    from edasketch import model
    from edasketch.assim import MemberProblem
    from edasketch.covariance import DiagonalNoise, GridCovFactor
    from edasketch.obs import ObsNetwork, strided_grid
    from edasketch.streams import substream
    n, N = cfg.n, cfg.n_steps
    ub = GridCovFactor(n, cfg.sigma_bg, 1.0, 1)
    ub.symbol = _gaussian_symbol(n, cfg.sigma_bg, cfg.cov_length)
    rn = DiagonalNoise(cfg.sigma_obs)
    net = ObsNetwork(strided_grid(n, n // cfg.obs_stride), list(cfg.obs_times))
    truth_traj = model.integrate(truth, cfg.dt, N, cfg.forcing)
    y = net.observe(truth_traj) + rn.apply(substream(cfg.seed, "obsnoise").standard_normal(net.p))
    x_bg = truth + ub.apply(substream(cfg.seed, "bg", 0).standard_normal(n))
    xj = x_bg + ub.apply(substream(cfg.seed, "bg", j).standard_normal(n))
    yj = y + rn.apply(substream(cfg.seed, "obsnoise", j).standard_normal(net.p))
    tj = model.integrate(xj, cfg.dt, N, cfg.forcing)
    return MemberProblem(tj, net, ub, rn, yj - net.observe(tj))


def _cpu_worker(args):
    """One host core: LMP-PCG iterations of one member with its own
    trajectory, J traced via quadratic_cost as in harness._solve_with_lmp
    (harness.py:178-182).  kind "reference": the unmodified edasketch
    (MemberProblem.hessian_apply, krylov.pcg, lmp.SpectralLmp); kind "port":
    the oracle restatement (bit-identical algorithm)."""
    cfg_id, j, iters, truth, kind = args
    from oracle.twin import BASELINE_CONFIGS
    cfg = BASELINE_CONFIGS[cfg_id]
    if kind == "reference":
        from edasketch.krylov import SolverConfig, pcg
        from edasketch.lmp import SpectralLmp
        prob = _ref_member(cfg, j + 1, truth)
    else:
        from oracle import l96
        from oracle.algorithms import SolverConfig, SpectralLmp, pcg
        from oracle.problem import MemberProblem
        from oracle.twin import baseline_inputs
        inp = baseline_inputs(cfg, members=j + 1, truth=truth)
        traj = l96.integrate(inp.member_x0[j], cfg.dt, cfg.n_steps, cfg.forcing)
        d = inp.member_y[j] - inp.net.observe(traj)
        prob = MemberProblem(traj, inp.net, inp.ub, inp.rn, d)
    # an orthonormal rank-k LMP: its apply costs what the control-built one
    # does (two n x k passes per application, lmp.py:62-74)
    rng = np.random.default_rng(j)
    k = min(cfg.k, cfg.n)  # cfg2: k = 50 > n = 40 keeps 40 pairs, as nystrom_evd does
    s, _ = np.linalg.qr(rng.standard_normal((cfg.n, k)))
    lmp = SpectralLmp(s, np.sort(rng.uniform(0, 1e3, k))[::-1], 2.0)
    b = prob.rhs()
    t0 = time.perf_counter()
    pcg(prob.hessian_apply, b, SolverConfig(max_iters=iters), precond=lmp,
        cost_fn=prob.quadratic_cost)
    return time.perf_counter() - t0, iters


def cpu_truth(cfg_id):
    """Spun-up truth (2000 RK4 steps): the reference's own model.rk4_step
    when baseline/_ref is present, else the oracle's (bit-identical)."""
    from oracle.twin import BASELINE_CONFIGS
    cfg = BASELINE_CONFIGS[cfg_id]
    if reference_available():
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        from edasketch import model
        x = np.full(cfg.n, cfg.forcing)
        x[0] += 0.01
        for _ in range(cfg.spinup_steps):
            x = model.rk4_step(x, cfg.dt, cfg.forcing)
        return x
    from oracle import l96
    return l96.deterministic_truth(cfg.n, cfg.dt, cfg.forcing, cfg.spinup_steps)


def _pool_init(ref_dir):
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    if ref_dir and ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)


def cpu_sample(cfg_id, seconds, cores, truth, iters=None):
    """Bounded CPU sample: ``cores`` members, each running ``iters`` PCG
    iterations in its own process; returns (applies/s, busy s, iters, wall s,
    kind).  kind = "reference" when the unmodified reference is installed in
    baseline/_ref, else "port"."""
    from oracle.twin import BASELINE_CONFIGS
    cfg = BASELINE_CONFIGS[cfg_id]
    kind = "reference" if reference_available() else "port"
    if iters is None:
        # measured on a Xeon core: ~2e-7 s per element-step for
        # one LMP-PCG iteration with the J trace; each process runs ~seconds/4
        per_iter = 2.0e-7 * cfg.n * cfg.n_steps
        iters = int(max(2, min(cfg.pcg_iters, seconds / 4.0 / max(per_iter, 1e-5))))
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"  # one core per process; inherited by spawn
    ctx = mp.get_context("spawn")
    with ctx.Pool(cores, initializer=_pool_init, initargs=(REF_DIR if kind == "reference" else "",)) as pool:
        t0 = time.perf_counter()
        res = pool.map(_cpu_worker, [(cfg_id, j, iters, truth, kind) for j in range(cores)])
        wall = time.perf_counter() - t0
    busy = max(r[0] for r in res)
    applies = sum(r[1] for r in res)
    cpu_sample.per_core = sum(r[1] / r[0] for r in res) / len(res)  # one process = one core
    return applies / busy, busy, iters, wall, kind


def cpu_description(kind, cores, iters, cfg, busy, per_step=False):
    what = ("the UNMODIFIED reference edasketch (pip-installed into baseline/_ref): "
            "assim.MemberProblem.hessian_apply + quadratic_cost, krylov.pcg, lmp.SpectralLmp"
            if kind == "reference" else
            "the oracle port of edasketch (oracle/, a bit-exact restatement; baseline/_ref absent)")
    return (f"{'per step ' if per_step else ''}{cores} members x {iters} LMP-PCG iterations "
            f"(J traced every iteration) of {cfg.name}, one member per process on its own core, "
            f"{what}; busy {busy:.1f} s; value_1core = the mean single-process rate "
            f"(SURVEY 8d '1 core')")


# ------------------------------------------------------------ GPU leg -----
NCU_FILE = os.path.join(ROOT, "profiles", "r2_sweep_ncu.json")
SWEEP_SOURCES = ("l96.cu", "sweep_tile.cu", "sweep.cuh", "common.cuh")


def sweep_sources_sha():
    """Hash of the sweep kernels' sources: an ncu record taken on other
    sources is reported as stale."""
    import hashlib
    h = hashlib.sha256()
    for f in SWEEP_SOURCES:
        with open(os.path.join(ROOT, "paper_2605_23571_b200", "csrc", f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def ncu_record(cfg_name, kernel):
    """Per-config ncu figures of one sweep (profiles/r2_sweep_ncu.json,
    written by tools/sweep_ncu.py from an `ncu --metrics` capture of that
    config's member-block sweep): DRAM bytes per sweep and the executed
    fp64-pipe utilisation."""
    try:
        with open(NCU_FILE) as fh:
            rec = json.load(fh)
    except (OSError, ValueError):
        return None
    k = rec.get("configs", {}).get(cfg_name, {}).get(kernel)
    if k is None:
        return None
    out = dict(k)
    out["file"] = os.path.relpath(NCU_FILE, ROOT)
    out["stale"] = rec.get("sources_sha") != sweep_sources_sha()
    return out


def time_fn(torch, fn, reps):
    """Mean device time of fn() (CUDA events on the current stream)."""
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3


def kernel_roofline(torch, eng, reps, peaks, cfg_name):
    """Time the dominant kernels live (CUDA events on the launching stream)
    on the PCG block: AD sweep and TL sweep over all members."""
    ens = eng.members
    lin = ens.lin
    M, n, N, p = ens.M, lin.n, lin.n_steps, lin.p
    dev = lin.states.device
    V = torch.randn(M, n, dtype=torch.float64, device=dev)
    W = torch.randn(M, p, dtype=torch.float64, device=dev)
    out = {"k_ad": time_fn(torch, lambda: lin.ad_cols(W, ens.traj_of), reps),
           "k_tl": time_fn(torch, lambda: lin.tl_cols(V, ens.traj_of), reps)}
    # the binding roofline for per-member trajectories is HBM,
    # with algorithmic bytes = the stored-stage formulation (4 stages x 8 B
    # read per element-step per sweep, + 8 B/element of the swept vector in
    # or out); algorithmic flops TL 37 / AD 42 per element-step
    flops = {"k_ad": 42.0 * N * n * M, "k_tl": 37.0 * N * n * M}
    alg_bytes = 32.0 * N * n * M + 8.0 * n * M
    dom = max(out, key=out.get)
    t = out[dom]
    nlaunch = -(-N // 12) if N > 12 else 1  # window chunks of <= 12 steps (l96.cu SWEEP_CHUNK)
    gbs = alg_bytes / t / 1e9
    tflops = flops[dom] / t / 1e12
    rec = ncu_record(cfg_name, dom)
    return {
        "bound": "hbm",
        "kernel": f"{dom} ({'AD' if dom == 'k_ad' else 'TL'} sweep over the {M} member "
                  f"trajectories; one sweep = {nlaunch} window-chunk launches, figures per sweep)",
        "achieved": gbs,
        "peak": peaks["hbm_gbs"],
        "unit": "GB/s",
        "frac": gbs / peaks["hbm_gbs"],
        # dram__bytes_read.sum + dram__bytes_write.sum of the sweep's launches,
        # from this config's ncu capture (the file and its freshness are named)
        "traffic": None if rec is None else rec["dram_bytes"],
        "traffic_source": (None if rec is None else
                           f"{rec['file']} ({cfg_name} {dom}, ncu --metrics, "
                           f"{'STALE: other sweep sources' if rec['stale'] else 'same sweep sources'})"),
        "algorithmic_bytes": alg_bytes,
        "basis": "SURVEY.md 8d: stored-stage formulation, 32*N*n + 8*n B per column per sweep. "
                 "The kernel recomputes the RK4 stages from the states (8 B/elem-step read), "
                 "so its physical DRAM traffic ('traffic') is below the algorithmic bytes "
                 "and what actually binds it is the FP64 pipe (see 'fp64').",
        "peak_source": "hbm: MEASURED_PEAKS.json hbm_gbs; fp64: DFMA loop measured in this run",
        "launch_ms": t * 1e3,
        "launch_ms_other": {k: v * 1e3 for k, v in out.items() if k != dom},
        "fp64": {
            "algorithmic_flops": flops[dom],
            "achieved_tflops": tflops,
            "peak_tflops": peaks["dfma_tflops"],
            "frac": tflops / peaks["dfma_tflops"],
            "dmma_peak_tflops": peaks["dmma_tflops"],
            "executed_pipe_util_pct": None if rec is None else rec.get("fp64_pipe_pct"),
            "executed_pipe_util_source": None if rec is None else rec["file"],
        },
    }


def measure_peaks(torch, lib_mod):
    lib = lib_mod.lib()
    sink = torch.zeros(1, dtype=torch.float64, device="cuda")
    res = {}
    for name, fn, fl in (("dfma", "edak_peak_dfma", lambda it, b: 2.0 * 8 * it * 256 * b),
                         ("dmma", "edak_peak_dmma", lambda it, b: 512.0 * 8 * it * 8 * b)):
        iters, blocks = 4096, 148 * 8
        getattr(lib, fn)(sink.data_ptr(), 64, blocks, lib_mod.stream())
        torch.cuda.synchronize()
        best = 0.0
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            getattr(lib, fn)(sink.data_ptr(), iters, blocks, lib_mod.stream())
            e.record()
            torch.cuda.synchronize()
            best = max(best, fl(iters, blocks) / (s.elapsed_time(e) * 1e-3) / 1e12)
        res[name + "_tflops"] = best
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            res["hbm_gbs"] = float(json.load(fh)["hbm_gbs"])
        res["hbm_source"] = "MEASURED_PEAKS.json"
    except (OSError, KeyError, ValueError):
        res["hbm_gbs"] = 6650.0  # B200_PROFILING.md fallback
        res["hbm_source"] = "fallback (B200_PROFILING.md)"
    return res


def applies_per_pass(cfg, total_members):
    """Hessian-column applications per pass: ell sketch columns + one per
    member per PCG iteration (rhs sweeps are half-applies, not counted)."""
    return cfg.ell + total_members * cfg.pcg_iters


def time_passes(torch, eng, steps, warmup, barrier=None):
    """W untimed passes, then K timed back to back (CUDA events around the
    whole block); returns (seconds per pass, last result, launches/pass)."""
    from paper_2605_23571_b200 import _lib
    barrier = barrier or torch.cuda.synchronize
    res = None
    for _ in range(max(warmup, 3)):
        res = eng.run()
    barrier()
    n0 = _lib.launch_count()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        res = eng.run()
    e.record()
    barrier()
    return s.elapsed_time(e) * 1e-3 / steps, res, (_lib.launch_count() - n0) // steps


def per_config_line(torch, cid, args, peaks):
    """Value/roofline of another BASELINE config, measured in this process."""
    import gc
    from paper_2605_23571_b200.engine import EdaPass
    from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble
    cfg = BASELINE_CONFIGS[cid]
    dens = build_ensemble(cfg)
    eng = EdaPass(dens)
    t, res, launches = time_passes(torch, eng, args.steps, args.warmup)
    out = {"config": config_dict(cfg, 1), "value": applies_per_pass(cfg, cfg.members) / t,
           "unit": UNIT, "ms_per_step": t * 1e3, "steps": args.steps,
           "member_pcg_solves_per_s": cfg.members / t, "gpu_launches": int(launches)}
    if cfg.n >= 1024:
        out["roofline"] = kernel_roofline(torch, eng, args.kernel_reps, peaks, cfg.name)
        out["roofline"]["kernel_share_of_step"] = (out["roofline"]["launch_ms"] *
                                                   (cfg.pcg_iters + 2) / (t * 1e3))
    else:
        out["roofline"] = None
        out["roofline_note"] = ("n = 40: the whole batched solve is one persistent launch "
                                "(pcg_small.cu), latency-bound; no sweep kernel to roofline")
    del eng, dens, res
    gc.collect()
    torch.cuda.empty_cache()
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2605_23571_b200 import _lib, build
    build.build()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # EDAK_BENCH_FUNCTIONAL=1: functional check of the multi-rank code path
    # on a box with fewer GPUs (ranks share devices, gloo collectives); its
    # numbers are not measurements
    functional = os.environ.get("EDAK_BENCH_FUNCTIONAL") == "1"
    if functional:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if functional:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2605_23571_b200.engine import EdaPass
    from paper_2605_23571_b200.parallel import max_over_ranks, shard
    from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble
    cfg = BASELINE_CONFIGS[args.config]
    if args.scaling == "weak":
        offset, count, total = rank * cfg.members, cfg.members, cfg.members * world
    else:
        offset, count = shard(cfg.members, world, rank)
        total = cfg.members
    dens = build_ensemble(cfg, members=count, member_offset=offset)
    eng = EdaPass(dens, member_offset=offset, total_members=total, distributed=world > 1)
    applies = applies_per_pass(cfg, total)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(max(args.warmup, 3)):
        res = eng.run()
    barrier()
    n0 = _lib.launch_count()
    barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_host0 = time.perf_counter()
    s.record()
    for _ in range(args.steps):
        res = eng.run()
    e.record()
    barrier()
    t_host1 = time.perf_counter()
    launches = (_lib.launch_count() - n0) // args.steps
    local_s = s.elapsed_time(e) * 1e-3
    clk = clocks.stop(t_host0, t_host1)
    t_step = max_over_ranks(local_s, torch.device("cuda", local)) / args.steps
    value = applies / t_step

    # ---- e2e: the same pass from HOST inputs, through the public API.  Per
    # step the host ships each row's initial state (x_b, x_j) and its
    # (perturbed) observations y_j (pinned -> device); the device integrates
    # the trajectories, forms the innovations (DeviceEnsemble.refresh,
    # eda.py:99-105) and runs the pass; the increments x come back to the host.
    e2e = None
    if not args.no_e2e:
        h_x0 = torch.empty_like(dens.x0, device="cpu").pin_memory()
        h_x0.copy_(dens.x0)
        h_y = torch.empty_like(dens.y, device="cpu").pin_memory()
        h_y.copy_(dens.y)
        h_x = torch.empty((count, cfg.n), dtype=torch.float64).pin_memory()

        # the copies run on their own stream, double-buffered: step k+1's H2D
        # overlaps step k's solve and step k's D2H overlaps step k+1's start;
        # every step still moves all of its bytes inside the timed region
        cs = torch.cuda.Stream()
        main = torch.cuda.current_stream()
        d_x0 = [torch.empty_like(dens.x0) for _ in range(2)]
        d_y = [torch.empty_like(dens.y) for _ in range(2)]
        h2d_done = [torch.cuda.Event(), torch.cuda.Event()]
        consumed = [torch.cuda.Event(), torch.cuda.Event()]
        x_ready = torch.cuda.Event()

        def h2d(b):
            with torch.cuda.stream(cs):
                cs.wait_event(consumed[b])
                d_x0[b].copy_(h_x0, non_blocking=True)
                d_y[b].copy_(h_y, non_blocking=True)
                h2d_done[b].record(cs)

        def e2e_step(k):
            b = k & 1
            main.wait_event(h2d_done[b])
            dens.refresh(d_x0[b], d_y[b])
            consumed[b].record(main)
            h2d(b ^ 1)  # next step's inputs, while this one solves
            r = eng.run()
            x_ready.record(main)
            with torch.cuda.stream(cs):
                cs.wait_event(x_ready)
                # r.x was allocated on the main stream and r dies with this
                # step: keep its block out of the allocator until the copy ran
                r.x.record_stream(cs)
                h_x.copy_(r.x, non_blocking=True)
            return r

        for b in range(2):
            consumed[b].record(main)
        h2d(0)
        e2e_step(0)
        main.wait_stream(cs)
        barrier()
        s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s2.record()
        h2d(1)
        for k in range(args.steps):
            e2e_step(k + 1)
        main.wait_stream(cs)
        e2.record()
        barrier()
        t2 = max_over_ranks(s2.elapsed_time(e2) * 1e-3, torch.device("cuda", local)) / args.steps
        h2d = h_x0.numel() * 8 + h_y.numel() * 8
        d2h = h_x.numel() * 8 + 2 * count * (cfg.pcg_iters + 1) * 8 + 8 * count
        e2e = {"value": applies / t2, "unit": UNIT, "ms_per_step": t2 * 1e3,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "path": "host pinned x0 + y per row -> DeviceEnsemble.refresh (GPU RK4 "
                       "trajectories, innovations) -> EdaPass.run (C-ABI) -> host x; "
                       "copies on a second stream, double-buffered across steps"}

    roof, peaks = None, None
    if rank == 0:
        peaks = measure_peaks(torch, _lib)
        roof = kernel_roofline(torch, eng, args.kernel_reps, peaks, cfg.name)
        # the dominant sweep runs once per PCG iteration, once for the rhs
        # and once for the sketch: ~(iters + 2) launches per step
        roof["kernel_share_of_step"] = (roof["launch_ms"] * (cfg.pcg_iters + 2) /
                                        (t_step * 1e3))
    per_config = None
    if rank == 0 and world == 1 and args.per_config.strip():
        tr0 = res.traces[0]
        check = {"member0_J_first_last": [tr0.cost[0], tr0.cost[-1]],
                 "member0_resnorm_last": tr0.resnorm[-1],
                 "lmp_values_top": [float(v) for v in res.approx.values[:3]]}
        del eng, dens, res
        import gc
        gc.collect()
        torch.cuda.empty_cache()
        per_config = {}
        for cid in [int(c) for c in args.per_config.split(",") if c.strip()]:
            if cid != args.config:
                per_config[BASELINE_CONFIGS[cid].name] = per_config_line(torch, cid, args, peaks)
    elif rank == 0:
        tr0 = res.traces[0]
        check = {"member0_J_first_last": [tr0.cost[0], tr0.cost[-1]],
                 "member0_resnorm_last": tr0.resnorm[-1],
                 "lmp_values_top": [float(v) for v in res.approx.values[:3]]}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = len(os.sched_getaffinity(0))
        truth = cpu_truth(args.config)
        v, busy, iters, wall, kind = cpu_sample(args.config, args.cpu_seconds, cores, truth)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
               "value_1core": cpu_sample.per_core,
               "sample": cpu_description(kind, cores, iters, cfg, busy)}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": t_step * 1e3,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64", "data": f"synthetic (seeded BASELINE {cfg.name} twin experiment)",
            "config": config_dict(cfg, world, args.scaling),
            "member_pcg_solves_per_s": total / t_step,
            "applies_per_step": applies,
            "e2e": e2e, "roofline": roof, "cpu_baseline": cpu,
            "gpu_launches": int(launches),
            "clocks": clk,
            "peaks": peaks,
            "per_config": per_config,
            "check": check,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from oracle.twin import BASELINE_CONFIGS
    cfg = BASELINE_CONFIGS[args.config]
    cores = len(os.sched_getaffinity(0))
    truth = cpu_truth(args.config)
    if args.warmup > 0:
        cpu_sample(args.config, 1.0, cores, truth, iters=2)
    vals, walls, per_core = [], [], []
    iters, kind = None, None
    per_step = min(args.cpu_seconds, 150.0 / max(args.steps, 1))
    for _ in range(args.steps):
        v, busy, iters, wall, kind = cpu_sample(args.config, per_step, cores, truth, iters)
        vals.append(v)
        walls.append(busy)
        per_core.append(cpu_sample.per_core)
    value = float(np.median(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.median(walls)) * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded BASELINE {cfg.name} twin experiment)",
        "config": config_dict(cfg, world, args.scaling),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "value_1core": float(np.median(per_core)),
                         "sample": cpu_description(kind, cores, iters, cfg, float(np.median(walls)),
                                                   per_step=True)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
