"""Preconditioned CG on the GPU (mirrors reference ``krylov.py``).

``pcg`` keeps the reference signature and semantics (krylov.py:49-105):
x0 = 0, fixed iteration budget, optional residual_rtol, per-iteration trace
of cost J(x), preconditioned residual norm sqrt(max(r.z, 0)) and matvec
count, the same stop rules and the same RuntimeError messages.

``pcg_members`` is the batched engine: every ensemble member runs its own
PCG recurrence (no coupling, krylov.py:49-97 per member) but each step is
one launch over all members:

    Hp      edak_hessian_block   (member j's own trajectory, I + A fused,
                                  p.Hp tile partials in the last U_B pass)
    alpha   edak_pcg_alpha       (breakdown flag, x/r update, cost, |r|^2)
    beta    edak_pcg_lmp_beta    (W = S^T r; r.Pr = |r|^2 + W^T diag(c) W;
                                  stop test; p = r + beta p + S(c o W) in
                                  the DMMA GEMM epilogue -- z = P r is
                                  never materialised)

With a two-pass (non-orthonormal S) or user preconditioner the beta step is
z = P r (edak_lmp_apply / callable) then edak_pcg_beta (r.z, stop, p).

All reductions are fixed-order (deterministic).  The cost trace uses the J
identity J(x) = 1/2 x.(I+A)x - b.x + 1/2 d.R^-1 d (test_assim.py:52-63) with
(I+A)x = b - r, i.e. J(x_i) = J(0) - 1/2 x_i.(b + r_i): one fused dot in the
x/r update instead of a TL sweep per iteration (``cost="exact"`` re-evaluates
quadratic_cost with a TL sweep instead; tests hold the two to 1e-10).
Per-member status stays on the device; the host reads it once at the end
(or every ``check_every`` iterations when a residual tolerance can stop
members early).
"""

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev, _lib


@dataclass
class SolverConfig:
    """krylov.py:25-37."""

    max_iters: int = 40
    residual_rtol: float | None = None
    trace_cost: bool = True

    def __post_init__(self):
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")


@dataclass
class SolveTrace:
    """krylov.py:40-46."""

    iterations: list = field(default_factory=list)
    cost: list = field(default_factory=list)
    resnorm: list = field(default_factory=list)
    matvecs: list = field(default_factory=list)
    status: str = "max_iters"


class PcgBreakdown(RuntimeError):
    """Raised like the reference (RuntimeError); ``member`` names the column."""

    def __init__(self, msg, member=0):
        super().__init__(msg)
        self.member = member


def _traces(status, iters, hist_rz, hist_J, trace_cost):
    bad = np.flatnonzero(status >= 2)
    if bad.size:
        c = int(bad[0])
        if status[c] == 3:
            raise PcgBreakdown("preconditioner is not positive definite", c)
        raise PcgBreakdown(f"system matrix is not positive definite (iteration {int(iters[c])})", c)
    resn = np.sqrt(np.maximum(hist_rz, 0.0))
    out = []
    for c in range(status.shape[0]):
        last = int(iters[c])
        rng = list(range(last + 1))
        tr = SolveTrace(iterations=rng, matvecs=list(rng), resnorm=resn[c, : last + 1].tolist(),
                        cost=(hist_J[c, : last + 1].tolist() if trace_cost
                              else [float("nan")] * (last + 1)),
                        status="converged" if status[c] == 1 else "max_iters")
        out.append(tr)
    return out


class _PcgRun:
    """State and per-iteration launches of one batched PCG (pcg_device).
    Split out so that several independent member groups can be stepped in
    lockstep on their own CUDA streams (pcg_members ``groups``)."""

    def __init__(self, apply_h, B, cfg, apply_p=None, cost=None, dot_tiles=0, lmp=None,
                 Z0=None):
        self.apply_h, self.apply_p, self.cfg = apply_h, apply_p, cfg
        B = B.contiguous()
        self.B = B
        M, n = B.shape
        self.M, self.n = M, n
        dev = B.device
        self.L = L = cfg.max_iters + 1
        self.X, self.R, self.P = torch.empty_like(B), torch.empty_like(B), torch.empty_like(B)
        self.HP = torch.empty_like(B)
        self.work = torch.empty(int(_lib.lib().edak_pcg_work_doubles(n, M)),
                                dtype=torch.float64, device=dev)
        self.hist_rz = torch.zeros((M, L), dtype=torch.float64, device=dev)
        self.hist_J = torch.full((M, L), float("nan"), dtype=torch.float64, device=dev)
        self.status = torch.zeros(M, dtype=torch.int32, device=dev)
        self.iters = torch.zeros(M, dtype=torch.int32, device=dev)
        s = _lib.stream()
        if Z0 is None:
            Z0 = apply_p(B) if apply_p is not None else B
        _lib.call("edak_pcg_init", n, M, B.data_ptr(), Z0.data_ptr(), self.X.data_ptr(),
                  self.R.data_ptr(), self.P.data_ptr(), self.work.data_ptr(),
                  self.hist_rz.data_ptr(), L, self.status.data_ptr(), self.iters.data_ptr(), s)
        self.trace_cost = bool(cfg.trace_cost and cost is not None)
        self.rec = self.trace_cost and cost[0] == "recurrence"
        self.cost = cost
        if self.rec:
            D, sigma2 = cost[1].contiguous(), float(cost[2])
            _lib.call("edak_pcg_cost0", D.shape[1], M, D.data_ptr(), sigma2,
                      self.hist_J.data_ptr(), L, s)
        elif self.trace_cost:
            self.hist_J[:, 0] = cost[1](self.X)
        self.rtol = -1.0 if cfg.residual_rtol is None else float(cfg.residual_rtol)
        self.rzb = self.work[-3 * M:-M]
        self.dot_tiles = dot_tiles
        self.dotp = (torch.empty((M, dot_tiles), dtype=torch.float64, device=dev)
                     if dot_tiles > 0 else None)
        self.lmp = lmp
        if lmp is not None:
            S = lmp[0]
            self.lmpwork = torch.empty(int(_lib.lib().edak_lmp_work_doubles(n, S.shape[0], M)),
                                       dtype=torch.float64, device=dev)

    def step(self, it):
        n, M, L, s = self.n, self.M, self.L, _lib.stream()
        X, R, P, HP, work = self.X, self.R, self.P, self.HP, self.work
        self.apply_h(P, HP, self.dotp)
        _lib.call("edak_pcg_alpha", n, M, P.data_ptr(), HP.data_ptr(), X.data_ptr(),
                  R.data_ptr(), work.data_ptr(), self.status.data_ptr(), self.iters.data_ptr(),
                  it, self.B.data_ptr() if self.rec else None, _lib.ptr(self.dotp),
                  self.dot_tiles, s)
        if self.trace_cost and not self.rec:
            run = self.status == 0
            self.hist_J[:, it] = torch.where(run, self.cost[1](X), self.hist_J[:, it])
        hJ = self.hist_J.data_ptr() if self.rec else None
        if self.lmp is not None:
            S, coef = self.lmp
            _lib.call("edak_pcg_lmp_beta", n, S.shape[0], M, S.data_ptr(), coef.data_ptr(),
                      R.data_ptr(), P.data_ptr(), work.data_ptr(), self.lmpwork.data_ptr(),
                      self.rtol, self.hist_rz.data_ptr(), hJ, L, self.status.data_ptr(),
                      self.iters.data_ptr(), it, s)
        else:
            Zr = self.apply_p(R) if self.apply_p is not None else R
            _lib.call("edak_pcg_beta", n, M, Zr.data_ptr(), R.data_ptr(), P.data_ptr(),
                      work.data_ptr(), self.rtol, self.hist_rz.data_ptr(), hJ, L,
                      self.status.data_ptr(), self.iters.data_ptr(), it, s)

    def snapshot(self, it):
        M = self.M
        rz = self.rzb[(it & 1) * M:(it & 1) * M + M] if it else self.rzb[:M]
        return (it, self.X.clone(), self.R.clone(), self.P.clone(), rz.clone())

    def traces(self):
        return _traces(self.status.cpu().numpy(), self.iters.cpu().numpy(),
                       self.hist_rz.cpu().numpy(), self.hist_J.cpu().numpy(), self.trace_cost)


def pcg_device(apply_h, B, cfg, apply_p=None, cost=None, check_every=8, snapshots=None,
               dot_tiles=0, lmp=None):
    """Batched PCG on a (M, n) device block of right-hand sides.

    apply_h(P, out, dotp) writes (I + A) P into ``out``; when ``dot_tiles``
    > 0 it also writes the (M, dot_tiles) tile partials of P.out into
    ``dotp`` (else dotp is None).  ``lmp`` = (S, coef) of a single-pass LMP
    selects the fused beta step (then ``apply_p`` is only used for z0).
    apply_p(R) -> P R (None = identity).  cost: None, ("recurrence", D,
    sigma2) with innovations D (M, p), or ("exact", fn) with fn(X) -> (M,)
    J values.  ``snapshots`` (a list) receives device copies of
    (it, X, R, P, rz) after every iteration (parity tests: teacher forcing).
    Returns X (M, n) and a list of SolveTrace."""
    run = _PcgRun(apply_h, B, cfg, apply_p, cost, dot_tiles, lmp)
    if snapshots is not None:
        snapshots.append(run.snapshot(0))
    for it in range(1, cfg.max_iters + 1):
        run.step(it)
        if snapshots is not None:
            snapshots.append(run.snapshot(it))
        if run.rtol >= 0.0 and it % check_every == 0 and bool((run.status != 0).all()):
            break
    return run.X, run.traces()


def _device_problem(apply_h):
    owner = getattr(apply_h, "__self__", None)
    lin = getattr(owner, "lin", None)
    if lin is not None and getattr(apply_h, "__name__", "") == "hessian_apply":
        return owner
    return None


def pcg(apply_h, b, cfg, precond=None, cost_fn=None):
    """Drop-in for krylov.pcg (krylov.py:49-97).

    Fully on the device when ``apply_h`` is our MemberProblem.hessian_apply
    (and ``cost_fn`` its quadratic_cost, ``precond`` our SpectralLmp);
    otherwise user callables are invoked on host arrays each iteration
    while the recurrence itself still runs on the device."""
    b_np = not isinstance(b, torch.Tensor)
    n = int(np.asarray(b).shape[0]) if b_np else int(b.shape[0])
    Bc, _, _ = _dev.to_cols(b, n)
    prob = _device_problem(apply_h)

    if prob is not None:
        work = prob.lin.work(1)

        def apply_h_cols(P, out, dotp):
            prob.n_matvecs += 1
            prob.hessian_cols(P, 1.0, out, work, dotp)
    else:
        def apply_h_cols(P, out, gp):
            y = np.asarray(apply_h(P[0].cpu().numpy()), dtype=float)
            out.copy_(torch.from_numpy(y)[None])

    if precond is None:
        apply_p = None
    elif hasattr(precond, "apply_cols"):
        apply_p = precond.apply_cols
    else:
        fn = precond if callable(precond) else precond.apply

        def apply_p(R):
            return _dev.to_cols(np.asarray(fn(R[0].cpu().numpy()), dtype=float), n)[0]

    cost = None
    if cfg.trace_cost and cost_fn is not None:
        owner = getattr(cost_fn, "__self__", None)
        if prob is not None and owner is prob and cost_fn.__name__ == "quadratic_cost":
            cost = ("recurrence", prob._d, prob.lin.sigma2)
        else:
            cost = ("exact", lambda X: torch.tensor([float(cost_fn(X[0].cpu().numpy()))],
                                                    dtype=torch.float64, device=X.device))
    X, traces = pcg_device(apply_h_cols, Bc, cfg, apply_p, cost,
                           dot_tiles=prob.lin.dot_tiles() if prob is not None else 0)
    x = X[0].cpu().numpy() if b_np else X[0]
    return x, traces[0]


_SIDE_STREAMS = {}
GRAPH_MAX_ELEMS = 1 << 22  # members x n up to which pcg_members replays a CUDA graph


def _side_streams(count):
    """Persistent side streams (per device): the caching allocator keeps its
    blocks per stream, so fresh streams every pass would re-allocate the PCG
    state each time."""
    dev = torch.cuda.current_device()
    lst = _SIDE_STREAMS.setdefault(dev, [])
    while len(lst) < count:
        lst.append(torch.cuda.Stream())
    return lst[:count]


GROUPS_MAX_ELEMS = 1 << 23  # members x n up to which >= 64 members run as two staggered groups


def _default_groups(M, n=0):
    """Two member groups on two streams fill what one group's launches leave
    idle at cfg4 (200 x 16384: 71.9 vs 76.5 ms per pass); at cfg5 (256 x
    262144) every launch already fills the GPU and one group is faster
    (216.4 vs 219.4 ms, tools/ab_pass.py)."""
    import os
    g = os.environ.get("EDAK_PCG_GROUPS")
    if g is not None:
        return max(1, int(g))
    return 2 if M >= 64 and M * n <= GROUPS_MAX_ELEMS else 1


SMALL_MAX_N = 256  # rings up to which pcg_members runs the persistent one-CTA-per-member solve


def _small_ok(ens, lmp, precond):
    lin = ens.lin
    return (lin.n <= SMALL_MAX_N and lin.n >= 8 and lin.stage_mode == "recompute"
            and lin.p * 8 <= 64 * 1024 and (precond is None or lmp is not None)
            and (lmp is None or lmp[0].shape[0] <= SMALL_MAX_N))


def pcg_members_small(ens, B, cfg, lmp=None, cost="recurrence"):
    """The whole batched solve in ONE launch (edak_pcg_small): one CTA per
    member runs every iteration -- Hessian apply, recurrence, J identity,
    single-pass LMP -- with the ring in shared memory.  Same results as the
    per-iteration path up to summation order."""
    M, n = B.shape
    dev = B.device
    L = cfg.max_iters + 1
    X = torch.empty_like(B)
    # one device buffer (hist_rz | hist_J | status, iters) -> one host copy
    buf = torch.empty(2 * M * L + M, dtype=torch.float64, device=dev)
    hist_rz, hist_J = buf[:M * L].view(M, L), buf[M * L:2 * M * L].view(M, L)
    si = buf[2 * M * L:].view(torch.int32)
    trace = bool(cfg.trace_cost and cost == "recurrence")
    rtol = -1.0 if cfg.residual_rtol is None else float(cfg.residual_rtol)
    S, coef = (None, None) if lmp is None else (lmp[0].contiguous(), lmp[1].contiguous())
    _lib.call("edak_pcg_small", _lib.C.byref(ens.lin._P), ens.traj_of.data_ptr(), M, B.data_ptr(),
              ens.D.data_ptr() if trace else None, _lib.ptr(S), _lib.ptr(coef),
              0 if S is None else S.shape[0], cfg.max_iters, rtol, X.data_ptr(),
              hist_rz.data_ptr(), hist_J.data_ptr() if trace else None, L, si.data_ptr(),
              si[M:].data_ptr(), _lib.stream())
    ens.n_matvecs += cfg.max_iters
    h = buf.cpu().numpy()
    hs = h[2 * M * L:].view(np.int32)
    return X, _traces(hs[:M], hs[M:], h[:M * L].reshape(M, L), h[M * L:2 * M * L].reshape(M, L),
                      trace)


def pcg_members(ens, B, cfg, precond=None, cost="recurrence", snapshots=None, fused=True,
                groups=None, check_every=8, graph=None, small=None):
    """Batched PCG over all members of an ``Ensemble``: B (M, n) device
    right-hand sides (e.g. ens.rhs_all()).  cost: "recurrence", "exact" or
    None.  ``fused`` folds p.Hp into the Hessian's last pass and a
    single-pass LMP into the beta step.

    ``groups`` > 1 splits the members into that many independent batches,
    each stepped on its own CUDA stream in lockstep: members never interact,
    so the streams only share the GPU, and one group's sweeps fill the SMs
    the other leaves idle (the last partial wave of every sweep launch, the
    HBM-bound vector updates and the DMMA GEMMs).  Default: 2 for >= 64
    members while members x n <= 2^23 (cfg4), else 1 (cfg5: every launch
    fills the GPU on its own); EDAK_PCG_GROUPS overrides.

    ``graph`` (default: for members x n <= 2^22, when the iteration count is
    fixed -- no residual_rtol -- and the LMP is single-pass or absent) records the whole
    solve (init + every iteration on every group stream) as ONE CUDA graph
    the first time an ensemble sees this shape, and replays it afterwards
    with the new right-hand sides and LMP copied into its resident buffers:
    no per-kernel launch cost and no inter-kernel gaps.
    ``small`` (default: rings of n <= 256 in recompute mode) runs the
    whole solve as one persistent launch (pcg_members_small).
    Returns (X (M, n), [SolveTrace] * M)."""
    import os
    M = ens.M
    G = _default_groups(M, B.shape[1]) if groups is None else groups
    if M < 2:
        G = 1
    G = max(1, min(G, M))
    apply_p = precond.apply_cols if precond is not None else None
    lmp = precond.single_pass() if (fused and precond is not None) else None
    B = B.contiguous()
    if graph is None:
        env = os.environ.get("EDAK_PCG_GRAPH")
        # measured: graphs pay off where launches dominate (cfg1-3: -10..-25%
        # per pass) and, with the staggered member groups, still -1% at cfg4
        # (75.5 -> 74.7 ms); no change at cfg5 (20 long iterations)
        graph = (env != "0") if env is not None else (B.numel() <= GRAPH_MAX_ELEMS)
    graph = (graph and snapshots is None and cfg.residual_rtol is None and fused
             and (precond is None or lmp is not None) and cost in ("recurrence", None))
    if small is None:
        env = os.environ.get("EDAK_PCG_SMALL")
        small = (env != "0") if env is not None else True
    if (small and snapshots is None and fused and cost in ("recurrence", None)
            and _small_ok(ens, lmp, precond)):
        return pcg_members_small(ens, B, cfg, lmp, cost)
    Z0 = B
    if apply_p is not None:
        # z0 = P b per member group, so every member's LMP GEMMs are the
        # group-sized kernels of its later iterations (the same kernels, hence
        # the same bits, whatever the member count of the pass or the rank)
        Z0 = torch.empty_like(B)
        bounds = _group_bounds(M, G)
        for lo, hi in zip(bounds[:-1], bounds[1:]):
            apply_p(B[lo:hi], out=Z0[lo:hi])
    if graph:
        return _pcg_members_graph(ens, B, Z0, cfg, lmp, cost, G)
    runs, streams = _group_runs(ens, B, Z0, cfg, apply_p, lmp, cost, G, fused)
    main = streams[0]

    def snap(it):
        # every group's state after iteration it, members in order (the
        # groups are stepped on their own streams: wait for all of them)
        for g in range(1, G):
            main.wait_stream(streams[g])
        parts = [r.snapshot(it) for r in runs]
        snapshots.append((it,) + tuple(torch.cat([p[i] for p in parts], 0) for i in range(1, 5)))
        for g in range(1, G):
            streams[g].wait_stream(main)

    if snapshots is not None:
        snap(0)
    rtol = runs[0].rtol
    stagger = _stagger()
    for it in range(1, cfg.max_iters + 1):
        for g, run in enumerate(runs):
            if stagger and it == 1 and g > 0:
                streams[g].wait_stream(streams[g - 1])
            with torch.cuda.stream(streams[g]):
                run.step(it)
        if G > 1:
            ens.n_matvecs += 1  # one batched member apply per iteration
        if snapshots is not None:
            snap(it)
        if rtol >= 0.0 and it % check_every == 0:
            for g in range(1, G):
                main.wait_stream(streams[g])
            if all(bool((r.status != 0).all()) for r in runs):
                break
    for g in range(1, G):
        main.wait_stream(streams[g])
    if G == 1:
        return runs[0].X, runs[0].traces()
    return torch.cat([r.X for r in runs], 0), [t for r in runs for t in r.traces()]


def _stagger():
    """Group g > 0 starts its first iteration after group g-1's, so the
    lockstep groups run one group-iteration out of phase for the whole solve.
    Measured at cfg4 (tools/pass_breakdown.py): every pass in the fast mode
    (75.6 ms) instead of mostly the slow one (78.3 ms) when both groups start
    together.  EDAK_PCG_STAGGER=0 turns it off."""
    import os
    return os.environ.get("EDAK_PCG_STAGGER", "1") != "0"


def _group_bounds(M, G):
    """Member-group bounds on even offsets: the overlap-save U_B pairs columns
    (2c, 2c + 1), so even bounds keep every member's pairing (and bits)
    independent of the grouping and of an even sharding across ranks."""
    return [0] + [min(M, ((M * g // G) + 1) & ~1) for g in range(1, G)] + [M]


def _group_runs(ens, B, Z0, cfg, apply_p, lmp, cost, G, fused):
    """One _PcgRun per member group, each initialised on its own stream."""
    M = ens.M
    bounds = _group_bounds(M, G)
    main = torch.cuda.current_stream()
    streams = [main] + _side_streams(G - 1)
    runs = []
    for g in range(G):
        lo, hi = bounds[g], bounds[g + 1]
        sub = ens if G == 1 else ens.subset(lo, hi)
        if g:
            streams[g].wait_stream(main)
        with torch.cuda.stream(streams[g]):
            work = sub.lin.work(sub.M)

            def apply_h_cols(P, out, dotp, sub=sub, work=work):
                sub.a_apply_members(P, ident=1.0, out=out, work=work, dot_part=dotp)

            c = None
            if cfg.trace_cost and cost == "recurrence":
                c = ("recurrence", sub.D, sub.lin.sigma2)
            elif cfg.trace_cost and cost == "exact":
                c = ("exact", sub.cost_members)
            runs.append(_PcgRun(apply_h_cols, B[lo:hi], cfg, apply_p, c,
                                sub.lin.dot_tiles() if fused else 0, lmp, Z0[lo:hi]))
    return runs, streams


class _PcgGraph:
    """A captured batched solve with its resident input buffers."""

    def __init__(self, ens, B, Z0, cfg, lmp, cost, G):
        self.B = torch.empty_like(B)
        self.Z0 = torch.empty_like(B)
        self.lmp = None
        if lmp is not None:
            self.lmp = (torch.empty_like(lmp[0]), torch.empty_like(lmp[1]))
        self.load(B, Z0, lmp)
        main = torch.cuda.current_stream()
        self.cap = torch.cuda.Stream()
        self.cap.wait_stream(main)
        self.graph = torch.cuda.CUDAGraph()
        n0 = int(_lib.lib().edak_launch_count())
        # an eager warm-up on the capture stream sets every kernel's
        # attributes (cudaFuncSetAttribute is not capturable) and allocates
        # the group streams' pools; the capture then reuses the same buffers
        with torch.cuda.stream(self.cap):
            self._record(ens, cfg, cost, G)
        self.cap.synchronize()
        with torch.cuda.graph(self.graph, stream=self.cap):
            self.runs = self._record(ens, cfg, cost, G)
        self.nodes = int(_lib.lib().edak_launch_count()) - n0
        self.nodes //= 2  # warm-up + capture
        main.wait_stream(self.cap)
        self.G = G
        self.iters = cfg.max_iters

    def load(self, B, Z0, lmp):
        self.B.copy_(B)
        self.Z0.copy_(Z0)
        if lmp is not None:
            self.lmp[0].copy_(lmp[0])
            self.lmp[1].copy_(lmp[1])

    def _record(self, ens, cfg, cost, G):
        runs, streams = _group_runs(ens, self.B, self.Z0, cfg, None, self.lmp, cost, G, True)
        stagger = _stagger()
        for it in range(1, cfg.max_iters + 1):
            for g, run in enumerate(runs):
                if stagger and it == 1 and g > 0:
                    streams[g].wait_stream(streams[g - 1])
                with torch.cuda.stream(streams[g]):
                    run.step(it)
        cur = torch.cuda.current_stream()
        for g in range(1, G):
            cur.wait_stream(streams[g])
        return runs


def _pcg_members_graph(ens, B, Z0, cfg, lmp, cost, G):
    key = (tuple(B.shape), cfg.max_iters, cfg.trace_cost, cost, G,
           None if lmp is None else tuple(lmp[0].shape))
    cache = ens.__dict__.setdefault("_pcg_graphs", {})
    entry = cache.get(key)
    if entry is None:
        entry = _PcgGraph(ens, B, Z0, cfg, lmp, cost, G)
        cache[key] = entry
    else:
        entry.load(B, Z0, lmp)
    main = torch.cuda.current_stream()
    entry.graph.replay()
    _lib._GRAPH_LAUNCHES[0] += entry.nodes
    ens.n_matvecs += entry.iters
    runs = entry.runs
    if entry.G == 1:
        return runs[0].X.clone(), runs[0].traces()
    return torch.cat([r.X for r in runs], 0), [t for r in runs for t in r.traces()]


# ----------------------------------------------------------------- Lanczos --

def lanczos_eigs(apply_h, n, m, n_eigs, seed=0):
    """Leading Ritz values of a symmetric operator with residual bounds
    (krylov.py:116-168): Lanczos with full reorthogonalization (twice, as
    DMMA GEMMs over the device basis) and restarts on invariant subspaces.

    Fully device-resident when ``apply_h`` is our hessian_apply; the scalar
    recurrence decisions (restart test) read one norm per step on the host,
    like the reference.  Fresh vectors come from the reference's
    ``substream(seed, "lanczos")`` host stream; the Ritz problem of the
    tridiagonal matrix is solved by the device Jacobi SVD (it is SPD for the
    I + A operators this is used on; values are |Ritz values| otherwise)."""
    from .linalg import col_dots, gemm_nn, gemm_tn, svd_jacobi
    from .twin import substream
    m = min(m, n)
    if not 1 <= n_eigs <= m:
        raise ValueError("need 1 <= n_eigs <= m")
    dev = _dev.device()
    prob = _device_problem(apply_h)
    if prob is not None:
        work = prob.lin.work(1)

        def h(v):
            prob.n_matvecs += 1
            return prob.hessian_cols(v, 1.0, None, work)
    else:
        def h(v):
            y = np.asarray(apply_h(v[0].cpu().numpy()), dtype=float)
            return torch.from_numpy(y).to(dev)[None]

    rng = substream(seed, "lanczos")
    basis = torch.zeros((m, n), dtype=torch.float64, device=dev)

    def orth(v, j):
        if j == 0:
            return v
        neg = -torch.ones(j, dtype=torch.float64, device=dev)
        for _ in range(2):
            c = gemm_tn(basis[:j], v)              # (1, j): basis_i . v
            v = gemm_nn(basis[:j], c, bscale=neg, Cin=v, beta=1.0)
        return v

    def norm2(v):  # fixed-order device dot (edak_col_dots), one host read
        return float(np.sqrt(float(col_dots(v, v)[0])))

    def fresh(j):
        for _ in range(5):
            v = torch.from_numpy(rng.standard_normal(n)).to(dev)[None]
            v = orth(v, j)
            norm = norm2(v)
            if norm > 1e-8 * np.sqrt(n):
                return v / norm
        return None

    alphas, betas = np.zeros(m), np.zeros(m)
    block_end = {}
    basis[0] = fresh(0)[0]
    scale = 0.0
    j = 0
    while j < m:
        w = h(basis[j:j + 1])
        alphas[j] = float(col_dots(basis[j:j + 1], w)[0])
        w = w - alphas[j] * basis[j:j + 1]
        w = orth(w, j + 1)
        beta = norm2(w)
        scale = max(scale, abs(alphas[j]), beta)
        if j + 1 == m:
            block_end[j] = beta
            break
        if beta <= 1e-12 * max(scale, 1.0):
            block_end[j] = beta
            nxt = fresh(j + 1)
            if nxt is None:
                m = j + 1
                break
            basis[j + 1] = nxt[0]
        else:
            betas[j] = beta
            basis[j + 1] = w[0] / beta
        j += 1
    tri = np.diag(alphas[:m]) + np.diag(betas[: m - 1], 1) + np.diag(betas[: m - 1], -1)
    U, sig, _ = svd_jacobi(torch.from_numpy(np.ascontiguousarray(tri.T)).to(dev))
    theta = sig.cpu().numpy()[:n_eigs]
    s = U.cpu().numpy()  # row i = eigenvector i (descending)
    bounds = np.array([sum(abs(b * s[i, pos]) for pos, b in block_end.items())
                       for i in range(n_eigs)])
    return theta, bounds
