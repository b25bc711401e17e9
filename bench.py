"""Benchmark: BASELINE.json configs[1] (C2), the isolated 2D operator benchmark.

Mesh 64x64 squares -> 8192 triangular macro-elements, m=4 (16 sub-triangles),
p=3, FP64; uniform flow rho=1, v=(1,0.3), P=1/(1.4*0.2^2) plus seeded N(0,1e-2)
noise on every nodal conserved value; one Jacobian assembly, second-layer
condensation + batched LU of all macros, then trace-operator applies on seeded
N(0,1) trace vectors (default_rng(1)).  A "step" is one matrix-free apply of
the condensed trace operator over all 8192 macros.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Prints one JSON line (rank 0).  value = trace-operator DOF-applies/s (whole
job); the condensation metric (macro-elements condensed/s) and the assembly
rate ride along in the same line.  --impl reference times the CPU restatement
of the reference algorithm (oracle/, the reference is 3D-only and cannot run
C2) on the host cores, on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_CELLS, M_SUB, P_DEG = 64, 4, 3
SIGMA = 1e-2
METRIC = "trace-operator DOF-applies/s"


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------


def c2_discretization(n_cells=N_CELLS):
    from paper_2402_11361_b200.cases import UniformFlow2D
    from paper_2402_11361_b200.discretization import Discretization
    from paper_2402_11361_b200.mesh import build_square_mesh

    case = UniformFlow2D()
    disc = Discretization(build_square_mesh(case.domain, n_cells, M_SUB, periodic=(True, True)), P_DEG, case.params)
    return case, disc


def c2_slab_discretization(world, comm):
    """Weak scaling: a (64 N) x 64 periodic strip of unit cells (same h as C2);
    rank r owns the 64 x 64-cell slab r (8192 macros, exactly C2's per-GPU
    work) and exchanges halos with its two neighbours."""
    from paper_2402_11361_b200.cases import UniformFlow2D
    from paper_2402_11361_b200.dist import DistDiscretization
    from paper_2402_11361_b200.mesh import build_square_mesh

    case = UniformFlow2D()
    mesh = build_square_mesh(((0.0, 0.0), (float(world), 1.0)), (N_CELLS * world, N_CELLS), M_SUB,
                             periodic=(True, True))
    return case, DistDiscretization(mesh, P_DEG, case.params, comm=comm)


def c2_state(case, disc, seed=0):
    """Nodal state + N(0, sigma) noise (seed 0); owner-side trace copy."""
    X = disc.node_coords().reshape(-1, 2)
    u = case.state(X).reshape(disc.n_mac, disc.L, disc.ns)
    u = u + SIGMA * np.random.default_rng(seed).standard_normal(u.shape)
    return u, disc.owner_trace_from_nodes(u)


def algorithmic_bytes_per_macro(disc):
    """B_ref: the reference's stored-operator bytes per
    macro apply."""
    d, ns, nf, L, Lf, m, p = disc.dim, disc.ns, disc.nf, disc.L, disc.Lf, disc.mesh.m, disc.p
    nq = disc.rm.n_quad
    nqf = disc.rm.n_quad_face
    ltr = nf * Lf * ns
    return 8 * ((L * ns) ** 2 + 3 * nf * (Lf * ns) ** 2 + m**d * nq * d * d * ns * ns
                + nf * m ** (d - 1) * nqf * d * ns * ns + 2 * ltr + (1 + d * d + nf * d + 2 * nf)) + 4 * ltr


def apply_kernel_bytes(disc):
    """Algorithmic HBM bytes per launch of each apply kernel (split apply): the
    B_ref terms each kernel streams plus the hand-off vectors between them."""
    d, ns, nf, L, Lf, m = disc.dim, disc.ns, disc.nf, disc.L, disc.Lf, disc.mesh.m
    nq, nqf = disc.rm.n_quad, disc.rm.n_quad_face
    n, bs, ltr = L * ns, Lf * ns, nf * Lf * ns
    npad = n + (n & 1)
    from paper_2402_11361_b200 import _lib

    si_factor = int(_lib.lib().mhdg_packed_lu_size(n))
    wv, wf = m**d * nq * d * d * ns * ns, nf * m ** (d - 1) * nqf * d * ns * ns
    geom = 1 + d * d + nf * d + nf
    M = disc.n_mac
    return {
        "apply_pre": M * (8 * (2 * nf * bs * bs + wv + wf + ltr + npad + 2 * ltr + geom) + 4 * ltr),
        "apply_si": M * 8 * (si_factor + 2 * npad),
        "apply_post": M * 8 * (nf * bs * bs + wf + npad + 2 * ltr + ltr + nf),
        "face_reduce": disc.n_trace * (3 * 8 + 2 * 4),
    }


def condense_executed_flops_per_macro(disc):
    """Flops the condensation kernels execute per macro: the Schur GEMMs on the
    tensor cores (k_schur_mma) and the factorization: batched LU ((2/3) n^3,
    the default factor kind) or the explicit Gauss-Jordan inverse (2 n^3)."""
    from paper_2402_11361_b200 import condense as CD
    d, ns, nf, L = disc.dim, disc.ns, disc.nf, disc.L
    rm = disc.rm
    schur = 2 * (rm.n_loc * ns * ns) * (rm.n_quad * d) * L * rm.n_sub
    schur += 2 * (rm.n_loc_face * ns * ns) * (rm.n_quad_face * d) * L * nf * rm.n_tri
    return {"schur": schur, "factor": (2 if CD.FACTOR == "inverse" else 2.0 / 3.0) * (L * ns) ** 3}


def assembly_flops_per_macro(disc):
    """Algorithmic flops of the Jacobian assembly per macro: the reference's dense
    contractions (assembly.py:455-470 volume, 578-585 face) per quadrature point in
    their cheapest order -- W1 = A g (nloc ns^2 d), the flux-Jacobian term
    (nloc ns^2 d + (nloc ns)^2), SUPG W1^T tau W1 ((nloc ns)^2 ns), the DIRK/PTC SUPG
    mass term ((nloc ns)^2); faces: proj x K1 and proj x S ((nlf ns)^2 each) -- at
    2 flops per multiply-add.  Residual and pointwise-physics work is not counted."""
    d, ns, nf = disc.dim, disc.ns, disc.nf
    rm = disc.rm
    nl, nlf = rm.n_loc, rm.n_loc_face
    vol = 2 * (2 * nl * ns * ns * d + (nl * ns) ** 2 * (1 + ns + 1))
    face = 2 * 2 * (nlf * ns) ** 2
    return rm.n_sub * rm.n_quad * vol + nf * rm.n_tri * rm.n_quad_face * face


def condense_flops_per_macro(disc):
    """F_cond = 2 d L^3 ns^2 + (2/3) (L ns)^3."""
    d, L, ns = disc.dim, disc.L, disc.ns
    return 2 * d * L**3 * ns**2 + (2.0 / 3.0) * (L * ns) ** 3


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


def committed_traffic():
    """ncu dram__bytes_read.sum + dram__bytes_write.sum per launch, from the
    committed profiles (profiles/traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


# ---------------------------------------------------------------------------
# clocks sampling (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------


class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.5)  # let the sampler start before the timed region
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": float(np.median(loaded)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU legs (oracle restatement of the reference algorithm)
# ---------------------------------------------------------------------------


def cpu_apply_rate(n_cells, applies, threads):
    """DOF-applies/s of the CPU restatement on an n_cells^2 periodic sample of
    the C2 workload (same m, p, state distribution and context)."""
    from threadpoolctl import threadpool_limits

    import oracle.hdg_oracle as O

    case, disc = c2_discretization(n_cells)
    u, uhat = c2_state(case, disc)
    with threadpool_limits(threads):
        f = O.Fields(u, O.gradient_refresh(disc, u, uhat), uhat)
        blocks, _ = O.jacobian(disc, f, O.Ctx.steady(1.0))
        cond = O.condense(blocks)
        xs = np.random.default_rng(1).standard_normal((applies, disc.n_trace))
        cond.apply_trace(xs[0])
        t0 = time.perf_counter()
        for x in xs:
            cond.apply_trace(x)
        dt = time.perf_counter() - t0
    return disc.n_trace * applies / dt, disc, dt


def run_reference(args, rank):
    """CPU restatement of the reference algorithm on the host cores: setup once
    on a bounded C2 sample, each step one apply over the sample."""
    if rank != 0:
        return
    from threadpoolctl import threadpool_limits

    import oracle.hdg_oracle as O

    threads = len(os.sched_getaffinity(0))
    n_cells = 8
    case, disc = c2_discretization(n_cells)
    u, uhat = c2_state(case, disc)
    with threadpool_limits(threads):
        f = O.Fields(u, O.gradient_refresh(disc, u, uhat), uhat)
        blocks, _ = O.jacobian(disc, f, O.Ctx.steady(1.0))
        cond = O.condense(blocks)
        xs = np.random.default_rng(1).standard_normal((args.warmup + args.steps, disc.n_trace))
        for i in range(args.warmup):
            cond.apply_trace(xs[i])
        t0 = time.perf_counter()
        for i in range(args.steps):
            cond.apply_trace(xs[args.warmup + i])
        dt = time.perf_counter() - t0
    value = disc.n_trace * args.steps / dt
    sample = (f"C2 restatement (oracle/) on a {n_cells}x{n_cells} periodic sample ({disc.n_mac} macros, m=4, "
              f"p=3, {disc.n_trace} trace dofs), one apply per step; the per-DOF rate is intensive")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "DOF-applies/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2 2D operator benchmark (64x64x2 macros, m=4, p=3)", "global_batch": None,
                   "seq_len": None, "parallelism": "cpu"},
        "cpu_baseline": {"value": value, "unit": "DOF-applies/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "DOF-applies/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------


def fp64_gemm_peak(torch, n=8192, reps=5):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    torch.matmul(a, b)
    torch.cuda.synchronize()
    best = math.inf
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    del a, b
    torch.cuda.empty_cache()
    return 2.0 * n**3 / best / 1e12


def _max_over_ranks(dist, t):
    import torch

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    tt = torch.tensor([t], dtype=torch.float64, device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    return float(tt)


def run_gpu(args, rank, world):
    import torch

    from paper_2402_11361_b200 import _lib
    from paper_2402_11361_b200 import assembly as A
    from paper_2402_11361_b200.condense import CondensedSchur
    from paper_2402_11361_b200.dist import DistCondensed
    from paper_2402_11361_b200.device import current_stream

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % torch.cuda.device_count())
    dist = None
    if world > 1:
        import torch.distributed as dist  # noqa: F811

        # MHDG_DIST_BACKEND=gloo: functional check of the slab path with several
        # ranks on one GPU (host-staged halos; not a measurement)
        backend = os.environ.get("MHDG_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    L = _lib.lib()

    ddisc = None
    if world > 1:
        from paper_2402_11361_b200.dist import Comm

        case, ddisc = c2_slab_discretization(world, Comm())
        disc = ddisc.local
        u, uhat_local = c2_state(case, disc, seed=rank)
        uhat = uhat_local[: ddisc.n_trace]  # owned faces (side 0 is local on every owned face)
    else:
        case, disc = c2_discretization()
        u, uhat = c2_state(case, disc)
    dd = disc.device
    top = ddisc if ddisc is not None else disc  # the discretization the public API is called with
    fields = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
    uh_local = ddisc.forward(fields.uhat) if ddisc is not None else fields.uhat
    fields.q = A.gradient_refresh(disc, fields.u, uh_local)
    ctx = A.StageContext.steady(1.0)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    # ---- assembly (one Jacobian assembly, timed) ----
    torch.cuda.synchronize()
    blocks, _ = A.jacobian(top, fields, ctx)  # warm
    del blocks  # the timed call reuses the cached block storage instead of allocating 11.5 GB
    torch.cuda.synchronize()
    a0, a1 = ev(), ev()
    with _lib.Timeline(16) as tl_asm:
        a0.record()
        blocks, _ = A.jacobian(top, fields, ctx)
        a1.record()
        a1.synchronize()
    t_asm = a0.elapsed_time(a1) / 1e3
    t_asm_k = tl_asm.ms.get("assemble", 0.0) / 1e3

    # ---- condensation: Schur correction + batched LU, timed ----
    cond = CondensedSchur.allocate(blocks)  # this rank's macros (the slab when N > 1)
    api = DistCondensed(ddisc, cond) if ddisc is not None else cond
    status = dd.status_buffer()
    cond.refactor_async(status)
    torch.cuda.synchronize()
    c_times = []
    with _lib.Timeline(64) as tl_cond:
        for _ in range(3):
            c0, c1 = ev(), ev()
            c0.record()
            cond.refactor_async(status)
            c1.record()
            c1.synchronize()
            c_times.append(c0.elapsed_time(c1) / 1e3)
    A.raise_status(status, "condense")
    t_cond = float(np.median(c_times))
    cond_k = {k: tl_cond.ms[k] / tl_cond.counts[k] / 1e3 for k in ("schur", "factor", "pack") if k in tl_cond.ms}

    # ---- applies ----
    K, W = args.steps, args.warmup
    n_own = top.n_trace
    xs = torch.as_tensor(np.random.default_rng(1 + rank).standard_normal((K + W, n_own)), device="cuda")
    y = torch.empty(n_own, dtype=torch.float64, device="cuda")
    y_face = torch.empty(disc.n_trace, dtype=torch.float64, device="cuda")
    y_loc = torch.empty(dd.n_local_trace, dtype=torch.float64, device="cuda")
    st = current_stream()

    def apply_split(x):
        """One trace-operator apply; with slabs DistCondensed.apply_trace: forward halo
        in flight while the interior macros are applied, then the halo-adjacent ones,
        reverse halo summed in the face reduction."""
        if ddisc is not None:
            api.apply_trace(x, out=y)
            return
        _lib.check(L.mhdg_apply_trace_local(dd.c, blocks.c, cond._fac, _lib.ptr(x), _lib.ptr(y_loc), st), "apply")
        _lib.check(L.mhdg_face_reduce(dd.c, _lib.ptr(y_loc), _lib.ptr(y_face), st), "reduce")

    clk = Clocks(local).__enter__()
    for i in range(W):
        apply_split(xs[i])
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches0 = L.mhdg_launch_count()
    t0, t1 = ev(), ev()
    torch.cuda.synchronize()
    # every library kernel in the timed region is bracketed by CUDA events on its
    # own (this) stream: per-kernel averages for the roofline
    with _lib.Timeline(8 * K + 64) as tl_apply:
        t0.record()
        for i in range(K):
            apply_split(xs[W + i])
        t1.record()
        torch.cuda.synchronize()
    launches = L.mhdg_launch_count() - launches0
    clk.__exit__(None, None, None)
    t_apply = t0.elapsed_time(t1) / 1e3
    if dist:
        t_apply = _max_over_ranks(dist, t_apply)
    kern_s = {k: tl_apply.ms[k] / tl_apply.counts[k] / 1e3 for k in tl_apply.ms}
    local_kernels = [k for k in ("apply_pre", "apply_si", "apply_post", "apply_fused", "apply_generic") if k in kern_s]
    k_apply = sum(kern_s[k] for k in local_kernels)

    # ---- e2e through the public API with pinned host buffers ----
    # Every step copies its input vector host -> device, applies through the public call
    # (CondensedSchur / DistCondensed.apply_trace) and copies the result device -> host.
    # Double-buffered as a serving loop would run it: step i+1's H2D and step i's D2H run on
    # their own copy streams while step i's apply runs; the timed region spans all copies.
    ne = max(3, min(K, 20))
    xh = [torch.empty(n_own, dtype=torch.float64, pin_memory=True) for _ in range(ne + 1)]
    for i, h in enumerate(xh):
        h.copy_(xs[i % (K + W)].cpu())
    yh = [torch.empty(n_own, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    xd = [torch.empty_like(y) for _ in range(2)]
    yd = [torch.empty_like(y) for _ in range(2)]
    comp = torch.cuda.current_stream()
    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
    Ev = lambda: torch.cuda.Event()  # noqa: E731

    def e2e_run(steps):
        h2d_done, comp_done, d2h_done = [Ev(), Ev()], [Ev(), Ev()], [Ev(), Ev()]
        with torch.cuda.stream(h2d_s):
            xd[0].copy_(xh[0], non_blocking=True)
            h2d_done[0].record()
        for i in range(steps):
            b = i & 1
            comp.wait_event(h2d_done[b])
            if i >= 2:
                comp.wait_event(d2h_done[b])  # yd[b] still being read back from step i-2
            api.apply_trace(xd[b], out=yd[b])
            comp_done[b].record(comp)
            if i + 1 < steps:  # prefetch the next step's input into the other buffer
                with torch.cuda.stream(h2d_s):
                    if i >= 1:
                        h2d_s.wait_event(comp_done[1 - b])  # step i-1 has consumed xd[1-b]
                    xd[1 - b].copy_(xh[i + 1], non_blocking=True)
                    h2d_done[1 - b].record()
            with torch.cuda.stream(d2h_s):
                d2h_s.wait_event(comp_done[b])
                yh[b].copy_(yd[b], non_blocking=True)
                d2h_done[b].record()
        comp.wait_stream(d2h_s)
        comp.wait_stream(h2d_s)

    e2e_run(2)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = ev(), ev()
    e0.record()
    e2e_run(ne)
    e1.record()
    e1.synchronize()
    t_e2e = e0.elapsed_time(e1) / 1e3 / ne
    if dist:
        t_e2e = _max_over_ranks(dist, t_e2e)
    # the last step's result, read back inside the timed region, equals the device apply
    y_chk = api.apply_trace(torch.as_tensor(xh[ne - 1].numpy(), device="cuda"))
    e2e_ok = bool(torch.equal(y_chk.cpu(), yh[(ne - 1) & 1]))

    # ---- stored local operators (B_A representation, csrc/ahat.cu): formation + applies ----
    stored = None
    if ddisc is None and not args.no_stored:
        torch.cuda.synchronize()
        f0, f1 = ev(), ev()
        f0.record()
        at = cond.form_local_operators()
        f1.record()
        f1.synchronize()
        t_form = f0.elapsed_time(f1) / 1e3
        for i in range(W):
            cond.apply_trace(xs[i], out=y)
        torch.cuda.synchronize()
        s0, s1 = ev(), ev()
        with _lib.Timeline(4 * K + 16) as tl_st:
            s0.record()
            for i in range(K):
                cond.apply_trace(xs[W + i], out=y)
            s1.record()
            s1.synchronize()
        t_st = s0.elapsed_time(s1) / 1e3
        k_st = tl_st.ms["apply_ahat"] / tl_st.counts["apply_ahat"] / 1e3
        ltr = disc.nf * disc.Lf * disc.ns
        b_st = (8 * ltr * ltr + 12 * ltr) * disc.n_mac  # blocks + gathered x and indices + y_loc
        cond.ahat = None
        y_mf = cond.apply_trace(xs[0]).clone()
        cond.ahat = at
        y_st = cond.apply_trace(xs[0])
        rel = float((y_st - y_mf).abs().max() / y_mf.abs().max())
        stored = {"what": "per-macro condensed trace blocks A^{T_i} (B_A, SURVEY 8d), formed once per "
                          "condensation from ltr unit-trace local applies; apply = batched GEMV k_ahat_gemv + "
                          "face reduce. Not the headline (value is the matrix-free B_ref apply).",
                  "value": n_own * K / t_st, "unit": "DOF-applies/s", "ms_per_step": 1e3 * t_st / K,
                  "form_seconds": t_form,
                  "break_even_applies": t_form / max(1e-12, t_apply / K - t_st / K),
                  "kernel": "k_ahat_gemv", "avg_launch_s": k_st, "algorithmic_bytes_per_launch": b_st,
                  "achieved_gbs": b_st / k_st / 1e9,
                  "max_rel_diff_vs_matrix_free": rel}
        del at
        cond.ahat = None

    # ---- coupling-recompute representation (B_min): only the S factors
    # resident, the coupling blocks re-formed per window before each local apply ----
    recompute = None
    if ddisc is None and not args.no_stored:
        from paper_2402_11361_b200.condense import CondensedRecompute

        y_mf = cond.apply_trace(xs[0]).clone()
        torch.cuda.synchronize()
        m_before = torch.cuda.memory_allocated()
        rb = A.RecomputeBlocks(disc, fields, ctx, chunk=2048)
        rcond = CondensedRecompute.build(rb)  # warm-up build
        torch.cuda.synchronize()
        r0, r1 = ev(), ev()
        r0.record()
        rcond.refactor()
        r1.record()
        r1.synchronize()
        t_rbuild = r0.elapsed_time(r1) / 1e3
        m_res = torch.cuda.memory_allocated() - m_before
        for i in range(W):
            rcond.apply_trace(xs[i], out=y)
        kr = max(3, K // 5)
        with _lib.Timeline(64 * kr + 64) as tl_rc:
            r0.record()
            for i in range(kr):
                rcond.apply_trace(xs[W + i], out=y)
            r1.record()
            r1.synchronize()
        t_rc = r0.elapsed_time(r1) / 1e3 / kr
        y_rc = rcond.apply_trace(xs[0])
        n_l, ltr_l = disc.L * disc.ns, disc.nf * disc.Lf * disc.ns
        geo = 1 + disc.dim**2 + disc.nf * disc.dim + 2 * disc.nf
        recompute = {"what": "coupling-recompute representation (B_min: S factors + face preconditioner "
                             "resident; k_couplings re-forms the face blocks and dG/dq stashes of a window "
                             "of macros before the split apply kernels read them). Not the headline.",
                     "value": n_own / t_rc, "unit": "DOF-applies/s", "ms_per_step": 1e3 * t_rc,
                     "window_macros": rb.chunk,
                     "kernels_ms_per_step": {k: v / kr for k, v in tl_rc.ms.items()},
                     "build_seconds": t_rbuild, "build_includes": "window-wise Jacobian assembly + Schur + LU + "
                                                                  "face-preconditioner sums and inverses",
                     "resident_bytes": int(m_res),
                     "resident_bytes_matrix_free": int(sum(getattr(blocks, k).numel() for k in blocks.KEYS) * 8
                                                       + cond.lu.numel() * 8 + cond.perm.numel() * 4
                                                       + cond.scratch.numel() * 8 + cond.work.numel() * 8),
                     "B_min_bytes_per_macro": 8 * (n_l * n_l + 3 * ltr_l + n_l + geo) + 4 * ltr_l,
                     "bitwise_equal_matrix_free": bool(torch.equal(y_rc, y_mf))}
        del rcond, rb

    # ---- Krylov vector kernels and the block preconditioner ----
    krylov = None
    if ddisc is None:
        from paper_2402_11361_b200 import krylov as KR

        pre = KR.block_precond_build(cond)  # warm-up (first launch of the build kernel)
        del pre
        torch.cuda.synchronize()
        p0, p1 = ev(), ev()
        with _lib.Timeline(64) as tl_pb:
            p0.record()
            pre = KR.block_precond_build(cond)
            p1.record()
            p1.synchronize()
        n = n_own
        rows = 21  # an inner GMRES column at restart 20 (krylov.py:270-276)
        V = torch.as_tensor(np.random.default_rng(7).standard_normal((rows + 1, n)), device="cuda")
        for _ in range(2):
            KR._icgs_launch(V, rows - 1, V[rows])
            pre(V[0])
        torch.cuda.synchronize()
        with _lib.Timeline(8 * K + 16) as tl_kr:
            for i in range(K):
                KR._icgs_launch(V, rows - 1, V[rows])
                pre(V[i % rows])
            torch.cuda.synchronize()
        bs = disc.Lf * disc.ns
        nfc = disc.mesh.n_faces
        t_icgs = tl_kr.ms["icgs"] / tl_kr.counts["icgs"] / 1e3
        t_pa = tl_kr.ms["precond_apply"] / tl_kr.counts["precond_apply"] / 1e3
        b_icgs = 8 * n * (3 * rows + 5)  # V_j streamed 3x; w read 3x, written 2x
        b_pa = 8 * (nfc * bs * bs + 2 * n)
        krylov = {"what": "one ICGS Arnoldi orthogonalisation (mhdg_icgs: 3 fused deterministic passes) "
                          "against 21 basis vectors and one block-preconditioner apply, C2 trace vectors",
                  "icgs": {"avg_launch_s": t_icgs, "rows": rows, "algorithmic_bytes": b_icgs,
                           "achieved_gbs": b_icgs / t_icgs / 1e9},
                  "precond_apply": {"avg_launch_s": t_pa, "algorithmic_bytes": b_pa, "achieved_gbs": b_pa / t_pa / 1e9},
                  "precond_build": {"seconds": p0.elapsed_time(p1) / 1e3,
                                    "kernel_seconds": tl_pb.ms.get("precond_build", 0.0) / 1e3,
                                    "faces": nfc, "block": bs,
                                    "flops": nfc * 2.0 * bs**3,
                                    "how": "register-tile Gauss-Jordan sweep of each symmetrised face block "
                                           "(bs^3 multiply-adds per face, csrc/precond.cu)"}}
        del V, pre

    peaks = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    fp64 = fp64_gemm_peak(torch) if rank == 0 else None
    b_mac = algorithmic_bytes_per_macro(disc)
    achieved_local = b_mac * disc.n_mac / k_apply / 1e9
    traffic = committed_traffic()
    kbytes = apply_kernel_bytes(disc)
    kernels = {}
    for k, sec in kern_s.items():
        entry = {"avg_launch_s": sec, "launches_per_step": tl_apply.counts[k] / K}
        if k in kbytes:
            gbs = kbytes[k] / sec / 1e9
            entry.update({"algorithmic_bytes_per_launch": kbytes[k], "achieved_gbs": gbs, "frac": gbs / hbm})
        kernels[k] = entry
    dom = max(kern_s, key=kern_s.get)  # dominant kernel by time
    from paper_2402_11361_b200 import condense as CD
    lu = CD.FACTOR == "lu"
    dom_name = {"apply_si": "k_lu_warp<2,4,3> (packed-LU forward/back substitution)" if lu
                else "k_si_stream<2,4,3> (TMA-streamed S^-1 apply)",
                "apply_pre": "k_apply_stream<2,4,3,pre>", "apply_post": "k_apply_stream<2,4,3,post>",
                "apply_fused": "k_apply_stream<2,4,3,fused>", "apply_generic": "k_apply_local<2>"}.get(dom, dom)
    dom_bytes = kbytes.get(dom, b_mac * disc.n_mac)
    achieved = dom_bytes / kern_s[dom] / 1e9
    f_mac = condense_flops_per_macro(disc)
    f_asm = assembly_flops_per_macro(disc)
    cond_tf = f_mac * disc.n_mac / t_cond / 1e12
    fx = condense_executed_flops_per_macro(disc)
    exec_tf = (fx["schur"] + fx["factor"]) * disc.n_mac / t_cond / 1e12

    n_dofs_job = world * n_own if ddisc is None else ddisc.global_mesh.n_faces * disc.Lf * disc.ns
    value = n_dofs_job * K / t_apply
    line = {
        "metric": METRIC, "value": value, "unit": "DOF-applies/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": 1e3 * t_apply / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2 2D operator benchmark: 64x64 squares -> 8192 triangular macros, m=4, p=3, "
                               "periodic, uniform flow + N(0,1e-2), StageContext.steady(pseudo_dt=1)",
                   "n_macros": disc.n_mac * world, "n_trace_dofs": n_dofs_job, "macros_per_gpu": disc.n_mac,
                   "global_batch": None, "seq_len": None,
                   "parallelism": (f"slab{world} (({N_CELLS}*{world})x{N_CELLS} periodic strip, forward/reverse "
                                   "face halos over NCCL P2P)") if world > 1 else "single",
                   "l2": "inputs larger than L2 (each apply streams ~%.1f GB of operator data)"
                         % (b_mac * disc.n_mac / 1e9)},
        "roofline": {"kernel": dom_name, "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic.get(dom + "_dram_bytes_per_launch"),
                     "algorithmic_bytes_per_launch": dom_bytes, "avg_launch_s": kern_s[dom],
                     "share_of_step": kern_s[dom] / (t_apply / K),
                     "timing": "CUDA events around every library kernel on its stream (mhdg_timeline)",
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)"},
        "apply_local": {"what": ("pre + LU solve + post kernels" if lu else "pre + S^-1 stream + post kernels")
                                + " against B_ref (SURVEY 8d)",
                        "achieved": achieved_local, "unit": "GB/s", "frac": achieved_local / hbm,
                        "algorithmic_bytes_per_launch": b_mac * disc.n_mac, "seconds": k_apply,
                        "traffic": traffic.get("apply_local_dram_bytes_per_launch")},
        "apply_kernels": kernels,
        "condense": {"metric": "macro-elements condensed/s", "value": disc.n_mac / t_cond, "unit": "macros/s",
                     "seconds": t_cond, "kernels_s": cond_k, "flops_per_macro": f_mac,
                     "roofline": {"bound": "fp64", "achieved": cond_tf, "peak": fp64, "unit": "TFLOP/s",
                                  "frac": (cond_tf / fp64) if fp64 else None,
                                  "flops": "canonical F_cond = 2dL^3ns^2 + (2/3)(L ns)^3 (SURVEY 8d)",
                                  "peak_source": "cuBLAS DGEMM 8192^3 measured in this run"},
                     "executed": {"flops_per_macro": fx, "achieved_tflops": exec_tf,
                                  "frac": (exec_tf / fp64) if fp64 else None,
                                  "note": "factor kind %s: " % CD.FACTOR
                                          + ("batched LU with partial pivoting, (2/3) n^3 (the F_cond term)" if lu
                                             else "explicit S^-1 (the reference's np.linalg.inv), 2 n^3")}},
        "assembly": {"metric": "macro-elements assembled/s (Jacobian + residual)", "value": disc.n_mac / t_asm,
                     "seconds": t_asm, "kernel_seconds": t_asm_k,
                     "roofline": {"bound": "fp64", "flops_per_macro": f_asm,
                                  "achieved": f_asm * disc.n_mac / t_asm_k / 1e12 if t_asm_k else None,
                                  "peak": fp64, "unit": "TFLOP/s",
                                  "frac": (f_asm * disc.n_mac / t_asm_k / 1e12 / fp64) if (fp64 and t_asm_k) else None,
                                  "flops": "the reference's Jacobian contractions (assembly.py:455-470, 578-585) "
                                           "in their cheapest order, per quadrature point"}},
        "krylov": krylov,
        "apply_stored": stored,
        "apply_recompute": recompute,
        "e2e": {"value": n_dofs_job / t_e2e, "unit": "DOF-applies/s", "steps": ne, "result_checked": e2e_ok,
                "how": "public apply_trace call per step with H2D of its input and D2H of its result, "
                       "double-buffered on two copy streams (next input and previous result overlap "
                       "the apply); all copies inside the CUDA-event timed region",
                "h2d_bytes_per_step": 8 * n_dofs_job, "d2h_bytes_per_step": 8 * n_dofs_job},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if stored is not None:
        stored["frac"] = stored["achieved_gbs"] / hbm
        stored["traffic"] = traffic.get("apply_ahat_dram_bytes_per_launch")
    if rank == 0 and not args.no_cpu_baseline:
        v, sdisc, dt = cpu_apply_rate(8, 10, 1)
        line["cpu_baseline"] = {"value": v, "unit": "DOF-applies/s", "cores": 1, "kind": "port",
                                "sample": f"oracle restatement, 8x8 periodic C2 sample ({sdisc.n_mac} macros, "
                                          f"{sdisc.n_trace} dofs), 10 applies in {dt:.1f} s, 1 thread"}
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-stored", action="store_true", help="skip the stored-operator (B_A) side measurement")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    run_gpu(args, rank, world)


if __name__ == "__main__":
    main()
