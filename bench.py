"""Benchmark of the per-stage HPS solve path (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

A *step* is one ESDIRK4 (ARK4(3)6L[2]SA) time step of the configured problem
through the drop-in ``TimeStepper`` -- 5 implicit HPS stage solves plus the
device stage right-hand-side assembly -- with the state resident in HBM.
``value`` = DOF*stages/s = N_dof * 5 * K / (device time of K steps, max over
ranks).  With N > 1 GPUs (torchrun) one problem is subtree-sharded over the
ranks; the ensemble config shards members; ``--shard
replicas`` runs one replica per GPU instead.

``e2e`` is the same metric through the public API with host-resident states:
every step copies its input state in from pinned host memory and its result
back out (``TimeStepper.step_host``; independent requests on the same input,
so one step's copies overlap its neighbours' compute).  ``e2e_dependent``:
a trajectory whose every step starts from the previous step's host result
(copies serialised with the compute).

``kernels``: per-kernel CUDA-event durations of the step's kernels (a
separate pass of eager steps with every launch bracketed by events,
``hps_ktimer_*``), each with its share of the step and its algorithmic HBM
bytes per launch.  ``roofline`` is
the dominant kernel's entry; ``traffic`` is its ncu dram bytes per launch from
the committed capture (profiles/traffic_kernels.json).  ``solve`` keeps the
whole-solve figures (plain solve, CUDA graph).

``parity``: the bench checks its own output -- C2's final state against the
manufactured solution, and one GPU step of the 64x64-leaf sample against the
CPU oracle's step from the same initial state (north-star bar 1e-10).

``cpu_baseline`` times the CPU oracle port (numpy/scipy, all host cores) on a
bounded sample: the 64x64-leaf version of the problem (same p, dt), one step,
build excluded.  ``--impl reference`` times the oracle port on the full
configuration (C2: 128x128 leaves, p=16), build outside the timed region, on
all host cores (the reference is pure Python and does not travel to the GPU
box).
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HPS stage solves/sec (DOF·stages/s), 2D ESDIRK4 fp64; % of HBM roofline"
UNIT = "DOF*stages/s"
TWO_PI = 2 * np.pi

# BASELINE.json configs (single-GPU workloads); C2 is the metric's config
CONFIGS = {
    "C1": dict(name="C1", n=8, p=12, dt=1e-3, kind="heat", k=1),
    "C2": dict(name="C2", n=128, p=16, dt=1e-4, kind="heat", k=1),
    "C3": dict(name="C3", n=256, p=12, dt=1e-3, kind="allen_cahn", k=1),
    "C4": dict(name="C4", n=512, p=10, dt=1e-5, kind="burgers_var", k=1),
    "C5": dict(name="C5", n=128, p=16, dt=1e-4, kind="ensemble", k=64),
}
SAMPLE_N = 64      # CPU sample: the 64x64-leaf subtree of the configured problem


def phi(pts):
    return np.sin(TWO_PI * pts[:, 0]) * np.sin(TWO_PI * pts[:, 1])


def sine_modes(seed, k=None, mmax=8, nmax=4):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.0, 1.0, size=(mmax, nmax) if k is None else (k, mmax, nmax))


def sine_field(coef, pts):
    x, y = pts[:, 0], pts[:, 1]
    mmax, nmax = coef.shape[-2:]
    sx = np.stack([np.sin(m * np.pi * x) for m in range(1, mmax + 1)])
    sy = np.stack([np.sin(n * np.pi * y) for n in range(1, nmax + 1)])
    if coef.ndim == 2:
        return np.einsum("mn,mp,np->p", coef, sx, sy)
    return np.einsum("kmn,mp,np->kp", coef, sx, sy)


def c4_fields():
    a = lambda x, y: 1 + 0.5 * np.sin(TWO_PI * x) * np.cos(TWO_PI * y)
    ax = lambda x, y: np.pi * np.cos(TWO_PI * x) * np.cos(TWO_PI * y)
    ay = lambda x, y: -np.pi * np.sin(TWO_PI * x) * np.sin(TWO_PI * y)
    return dict(c11=a, c22=a, c1=lambda x, y: -(ax(x, y) + 1.0), c2=lambda x, y: -(ay(x, y) + 0.5))


def make_problem(mod, cfg):
    """ParabolicProblem of the config for the package ``mod`` (ours or the
    oracle-facing description); returns (problem kwargs)."""
    kind = cfg["kind"]
    plain = cfg.get("plain", False)   # --plain-fields: the reference caller's numpy callables, undeclared g
    if kind == "heat":
        if plain:
            q = lambda t, pts: phi(pts) * (-np.sin(t) + 8 * np.pi ** 2 * np.cos(t))
            f = lambda t, pts: phi(pts) * np.cos(t)
        else:
            q = mod.SeparableField.product(phi, lambda t: -np.sin(t) + 8 * np.pi ** 2 * np.cos(t))
            f = mod.SeparableField.product(phi, np.cos)
        return dict(coeffs=mod.OperatorCoefficients(c11=1.0, c22=1.0), q=q, f=f,
                    u0=lambda pts: phi(pts))
    if kind == "allen_cahn":
        coef = sine_modes(0)
        g = lambda t, u, ux, uy: u - u ** 3
        return dict(coeffs=mod.OperatorCoefficients(c11=0.01, c22=0.01),
                    g=g if plain else mod.declare_nonlinear(g, ux=False, uy=False, pure=True),
                    u0=lambda pts: sine_field(coef, pts),
                    time_independent_bc=True)
    if kind == "burgers_var":
        coef = sine_modes(1)
        return dict(coeffs=mod.OperatorCoefficients(**c4_fields()),
                    g=mod.declare_nonlinear(lambda t, u, ux, uy: -u * ux, ux=True, uy=False, pure=True),
                    u0=lambda pts: sine_field(coef, pts),
                    time_independent_bc=True)
    if kind == "ensemble":
        coef = sine_modes(2, k=cfg["k"])
        q = mod.SeparableField.product(lambda pts: sine_field(coef, pts))
        return dict(coeffs=mod.OperatorCoefficients(c11=1.0, c22=1.0), q=q,
                    u0=lambda pts: np.zeros((cfg["k"], pts.shape[0])), time_independent_bc=True,
                    ncomp=cfg["k"])
    raise ValueError(kind)


def solve_bytes(tree, k, const_leaf):
    """Algorithmic HBM bytes of one stage solve; the root's
    Tstack is never applied (its flux has no consumer) and is not counted."""
    ni, nb, L = tree.ni, tree.nb, tree.L
    ops = 0
    vec = L * (2 * ni + 2 * nb)
    for d, lm in enumerate(tree.level_maps):
        c, n3, n12 = lm.count, lm.n3, lm.n12
        ops += c * (n3 * n3 + n3 * n12 + (n12 * n3 if d > 0 else 0))
        vec += c * (3 * n12 + 2 * n3)
    lam = 1 if const_leaf else L
    ops += lam * (ni * ni + ni * nb) + nb * ni
    return 8 * ops, 8 * k * vec


def solve_bytes_shared(tree, k):
    """HBM bytes of one stage solve with the shared (per-level) layout: one
    operator pair per level, the shared leaf operators, and the vectors."""
    ni, nb, L = tree.ni, tree.nb, tree.L
    ops = (ni * ni + ni * nb) + nb * ni + ni * nb
    vec = L * (2 * ni + 2 * nb)
    for d, lm in enumerate(tree.level_maps):
        n3, n12 = lm.n3, lm.n12
        ops += n3 * n3 + n3 * n12 + (n12 * n3 if d > 0 else 0)
        vec += lm.count * (3 * n12 + 2 * n3)
    return 8 * ops, 8 * k * vec


FP64_TFLOPS = 37.0   # measured DMMA peak on this pool's B200 (profiles/r01_fp64_peak.txt)


def solve_flops(tree, k, tensor_leaf=False):
    """FP64 flops of one stage solve as executed: the dense leaf products, or
    the tensor-product leaf solve (8 q^3 + 2 nb q per leaf) for the up pass."""
    ni, nb, L, q = tree.ni, tree.nb, tree.L, tree.q
    if tensor_leaf:
        e = L * (4 * q ** 3 + nb * q + ni * nb)
    else:
        e = L * (ni * ni + 2 * ni * nb)
    for d, lm in enumerate(tree.level_maps):
        e += lm.count * (lm.n3 * lm.n3 + lm.n3 * lm.n12 + (lm.n12 * lm.n3 if d > 0 else 0))
    return 2 * k * e


def level_shapes(n, p):
    """(count, n3, n12) of every parent level, root first, of an n x n-leaf
    tree with p nodes per leaf side (SURVEY.md 8(a) closed form: x-splits of
    m x m boxes have n3 = m q, n12 = 4 m q; y-splits of (m/2) x m boxes
    n3 = m q / 2, n12 = 3 m q)."""
    q = p - 2
    out, m, c = [], n, 1
    while m > 1:
        out.append((c, m * q, 4 * m * q))               # x-split of an m x m box
        out.append((2 * c, m * q // 2, 3 * m * q))      # y-split of an (m/2) x m box
        m //= 2
        c *= 4
    return out


def config_block(cfg):
    """The config dict both arms print (same workload)."""
    n, p = cfg["n"], cfg["p"]
    q = p - 2
    L, ni = n * n, q * q
    N = q * (p * L + 2 * n)
    ops = sum(n3 * n3 + 2 * n3 * n12 for _, n3, n12 in level_shapes(n, p)) * 8
    return {"workload": f"{cfg['name']}: {n}x{n} leaves, p={p}, {cfg['kind']}, ARK4 dt={cfg['dt']}, "
                        f"k={cfg['k']}, one ARK4 step per bench step (5 stage solves)"
                        + (", plain numpy field callables / undeclared g" if cfg.get("plain") else ""),
            "N_dof": N,
            "l2": ("inputs larger than L2, no flush (level operators streamed per stage solve %.2f GB "
                   "> 126 MB L2; state %.1f MB)" % (ops / 1e9, 8e-6 * N * cfg["k"])) if ops > 126e6 else
                  "working set fits the 126 MB L2 (a latency-bound configuration; no flush)"}


def kernel_bytes(shapes, dF, L, ni, nb, nbd, N, k=1, per_node=False):
    """Algorithmic HBM bytes per launch of the stage-path kernels
    (DESIGN.md): every vector byte a kernel must read or write once, every
    operator byte once per launch (shared layout: one operator per level;
    per_node: one per node, what the reference stores).  Up-level node: children's flux
    entries 2 n3 + n12 in, w3 n3 + flux n12 out, operator (n3 + n12) n3 (root
    n3 n3); down-level node: boundary values n12 + w3 n3 in, u3 n3 out,
    operator n3 n12 (root: precomputed by k_root_dir in the stage path).
    Returns {category: bytes or fn(nterms)}."""
    nops = (lambda c: c) if per_node else (lambda c: 1)

    def up(lv, root):
        c, n3, n12 = lv
        return 8 * (k * c * (3 * n3 + 2 * n12 - (n12 if root else 0)) + nops(c) * (n3 + (0 if root else n12)) * n3)

    def dn(lv, root):
        c, n3, n12 = lv
        return 8 * (k * c * (n12 + 2 * n3) + (0 if root else nops(c) * n3 * n12))

    wide = range(0, dF)
    fused = range(dF, len(shapes))
    c0, n3r, n12r = shapes[0]
    return {
        "k_mega": sum(up(shapes[d], d == 0) + dn(shapes[d], d == 0) for d in wide),
        "k_sub_up": sum(up(shapes[d], False) for d in fused) + 8 * k * L * nb,
        "k_sub_down": sum(dn(shapes[d], False) for d in fused),
        # leaf up: the stage terms in, the formed body load and the leaf fluxes out, Dirichlet data
        "leaf_up_terms": lambda nt: 8 * k * ((nt + 1) * L * ni + L * nb + nbd),
        # leaf down: body load + boundary values in, u_int and the L u history out
        "leaf_down": 8 * k * (L * ni + L * nb + 2 * L * ni),
        "leaf_lu": 8 * k * (L * ni + L * nb + L * ni),
        # the root's Dirichlet product of ns boundary-data rows: S_root once
        "root_dir": lambda ns: 8 * (n3r * n12r + ns * (n12r + n3r)),
        "combine_bnd": lambda nt: 8 * k * (nt + 1) * N,
    }


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()   # nvidia-smi takes a while to start: wait for its first row
            while not self.rows and time.time() - t0 < 5.0:
                time.sleep(0.02)
            self.n0 = len(self.rows)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc is not None:
            t0 = time.time()   # at least one row from inside / right at the end of the region
            while len(self.rows) <= self.n0 and time.time() - t0 < 1.0:
                time.sleep(0.02)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def _kernels_per_step(st, state):
    """Kernels one step launches (host-side count of an eager step)."""
    from paper_2306_02526_b200 import _lib
    lib = _lib.load()
    import torch
    n0 = lib.hps_launch_count()
    st._advance(state)
    torch.cuda.synchronize()
    return lib.hps_launch_count() - n0


def _time_solves(st, n, sharded=False):
    """CUDA-event time of one stage solve (the stepper's body load, boundary
    data and operators), replayed as a CUDA graph like inside the step.  A
    subtree-sharded solve (collectives inside) is timed eagerly, every rank
    in lockstep."""
    import torch
    k = st._k
    r = st._bufs.get("r")
    out = torch.empty((k, st.tree.N), dtype=torch.float64, device="cuda")
    fb = st._bc(0.0)
    if sharded:
        st._solve(st.ops, fb, r, out)
        torch.cuda.synchronize()
        times = []
        for _ in range(n):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            st._solve(st.ops, fb, r, out)
            e1.record()
            times.append((e0, e1))
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in times]
    from paper_2306_02526_b200.solver import graph_workspace
    with graph_workspace("bench-solve"):     # the graph's workspace, allocated by the warm solve
        st.ops.solve_device(fb, r, out)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            st.ops.solve_device(fb, r, out)
    g.replay()
    torch.cuda.synchronize()
    times = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        times.append((e0, e1))
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in times]


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def profiled_traffic(config):
    """dram bytes per solve from a committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(config)
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------

def oracle_stepper(cfg, n=None, record=False):
    """The CPU oracle's stepper of the config (n x n leaves; default the
    config's own n): (tree, stepper, initial state).  Checker / CPU baseline only."""
    from oracle import hps_oracle as O  # checker / CPU baseline only
    n = cfg["n"] if n is None else n
    tree = O.OTree(((0.0, 1.0), (0.0, 1.0)), n, n, cfg["p"])
    kind = cfg["kind"]
    kw = {}
    if kind == "heat":
        kw = dict(q=lambda t, pts: phi(pts) * (-np.sin(t) + 8 * np.pi ** 2 * np.cos(t)),
                  f=lambda t, pts: phi(pts) * np.cos(t))
        coeffs, u = O.OCoeffs(c11=1.0, c22=1.0), phi(tree.points)
    elif kind == "allen_cahn":
        coeffs = O.OCoeffs(c11=0.01, c22=0.01)
        kw = dict(g=lambda t, u, ux, uy: u - u ** 3)
        u = sine_field(sine_modes(0), tree.points)
    elif kind == "burgers_var":
        coeffs = O.OCoeffs(**c4_fields())
        kw = dict(g=lambda t, u, ux, uy: -u * ux)
        u = sine_field(sine_modes(1), tree.points)
    else:
        coeffs = O.OCoeffs(c11=1.0, c22=1.0)
        coef = sine_modes(2, k=cfg["k"])
        kw = dict(q=lambda t, pts: sine_field(coef, pts), ncomp=cfg["k"])
        u = np.zeros((cfg["k"], tree.N))
    st = O.OStepper(tree, coeffs, O.ark4_tableau(), cfg["dt"], record=record, **kw)
    return tree, st, u


def cpu_oracle_sample(cfg, steps, warmup, keep_state=False):
    """Times the oracle port on the SAMPLE_N x SAMPLE_N-leaf version of the
    config (build excluded).  keep_state: also return the state after the
    first step from the initial data (the GPU parity check)."""
    n = min(SAMPLE_N, cfg["n"])
    tree, st, u = oracle_stepper(cfg, n)
    t = 0.0
    first = None
    for _ in range(warmup):
        t, u = st.run(t, u, 1)
        first = u if first is None else first
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        t, u = st.run(t, u, 1)
        times.append(time.perf_counter() - t0)
        first = u if first is None else first
    k = cfg["k"]
    val = tree.N * k * 5 * len(times) / sum(times)
    sample = (f"{n}x{n}-leaf version of the config, p={cfg['p']}, k={k}, {len(times)} ARK4 step(s) "
              f"({5 * len(times)} stage solves + RHS), N={tree.N}, build excluded")
    if keep_state:
        return val, sample, times, first
    return val, sample, times


def run_reference(args, cfg, rank):
    """The reference arm: the CPU oracle port (a restatement of the reference
    hpstep algorithm; the reference itself is pure Python and cannot travel to
    the GPU box) on the FULL configuration -- C2: 128 x 128 leaves, p = 16,
    N = 3,673,600 -- with all host cores (numpy/scipy's OpenBLAS threads).
    The operator build is outside the timed region; W untimed steps, then K
    timed ARK4 steps from the configuration's initial data."""
    if rank != 0:
        return
    t0 = time.perf_counter()
    tree, st, u = oracle_stepper(cfg)
    build_s = time.perf_counter() - t0
    t = 0.0
    for _ in range(args.warmup):
        t, u = st.run(t, u, 1)
    times = []
    for _ in range(max(1, args.steps)):
        t1 = time.perf_counter()
        t, u = st.run(t, u, 1)
        times.append(time.perf_counter() - t1)
    k = cfg["k"]
    val = tree.N * k * 5 * len(times) / sum(times)
    cores = os.cpu_count()
    threads = os.environ.get("OPENBLAS_NUM_THREADS") or os.environ.get("OMP_NUM_THREADS") or str(cores)
    sample = (f"full configuration ({cfg['n']}x{cfg['n']} leaves, p={cfg['p']}, N={tree.N}), "
              f"{len(times)} timed ARK4 steps after {args.warmup} untimed, build {build_s:.1f} s excluded, "
              f"BLAS threads {threads}")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(cfg),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "build_s": build_s}
    if cfg["kind"] == "heat":
        uex = phi(tree.points) * np.cos(t)
        line["parity"] = {"manufactured_max_rel": float(np.abs(u - uex).max() / np.abs(uex).max()),
                          "manufactured_t": t}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--plain-fields", action="store_true",
                    help="q / f as plain numpy callables and g undeclared (the reference caller's code, "
                         "evaluated at cuts of the captured step)")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--layout", default=None, choices=[None, "auto", "per_node", "shared"],
                    help="operator storage (default: shared for constant coefficients)")
    ap.add_argument("--shard", default="auto", choices=["auto", "subtree", "replicas"],
                    help="N > 1 GPUs: subtree-shard one problem (auto) or run replicas")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config], plain=args.plain_fields)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args, cfg, rank)
        return

    import torch
    import torch.distributed as dist
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # HPSB_BENCH_DEVICE / HPSB_BENCH_BACKEND: exercise the multi-rank code path on
    # one GPU (gloo, host-staged exchanges) -- never for reported numbers
    local = int(os.environ.get("HPSB_BENCH_DEVICE", local))
    backend = os.environ.get("HPSB_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local)
    distributed = "TORCHELASTIC_RUN_ID" in os.environ or world > 1   # launched by torchrun
    if distributed:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    import paper_2306_02526_b200 as hb
    from paper_2306_02526_b200 import _lib
    from paper_2306_02526_b200.sharding import max_over_ranks as _max_over_ranks
    from paper_2306_02526_b200.sharding import ShardedTimeStepper, shard_problem

    lib = _lib.load()
    tree = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), cfg["n"], cfg["n"], cfg["p"])
    prob = hb.ParabolicProblem(**make_problem(hb, cfg))
    # ensembles shard by member; a single problem is subtree-sharded (both
    # strong scaling: fixed total work), or replicated with --shard replicas
    ensemble = prob.ncomp > 1
    subtree = world > 1 and not ensemble and args.shard != "replicas"
    if ensemble and world > 1:
        prob = shard_problem(prob, rank, world)
    scaling = "strong" if (ensemble or subtree) else "weak"
    t0 = time.perf_counter()
    if subtree:
        st = ShardedTimeStepper(tree, prob, "ARK4", dt=cfg["dt"], layout=args.layout)
    else:
        st = hb.TimeStepper(tree, prob, "ARK4", dt=cfg["dt"], layout=args.layout)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    k = prob.ncomp
    k_total = cfg["k"]
    state = st.initial_state()
    state = hb.StepperState(state.t, state.u_device)

    def barrier():
        torch.cuda.synchronize()
        if distributed:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        return _max_over_ranks(x, device="cuda")

    for _ in range(args.warmup):
        state = st.run(state, 1)
    barrier()
    n0 = lib.hps_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prof = os.environ.get("HPSB_PROFILE_RANGE") == "1"   # ncu --profile-from-start off
    with ClockSampler(local) as clk:
        if prof:
            torch.cuda.cudart().cudaProfilerStart()
        ev0.record()
        state = st.run(state, args.steps, check_every=max(1, args.steps))
        ev1.record()
        barrier()
        if prof:
            torch.cuda.cudart().cudaProfilerStop()
    launches = lib.hps_launch_count() - n0
    if launches == 0 and st._graph is not None:
        # graph replay: the library did not launch from the host; count the kernels of one step
        launches = _kernels_per_step(st, state) * args.steps
    ms = ev0.elapsed_time(ev1)
    ms = max_over_ranks(ms)
    copies = k_total if ensemble else (k if subtree else k * world)
    units = tree.N * 5 * args.steps * copies
    value = units / (ms * 1e-3)
    final = state

    # parity of the timed run itself: C2 / C1 have a manufactured solution
    parity = {}
    if cfg["kind"] == "heat" and not subtree:
        uf = final.u_device.reshape(-1)
        uex = torch.as_tensor(phi(tree.points) * np.cos(final.t), device=uf.device)
        parity["manufactured_max_rel"] = float((uf - uex).abs().max() / uex.abs().max())
        parity["manufactured_t"] = final.t

    # whole-solve figures (plain solve replayed as a graph) for reference
    solve_ms = _time_solves(st, 5 * args.steps, sharded=subtree)

    # per-kernel CUDA-event durations of the step (eager steps, every launch bracketed)
    kt_steps = 3
    kernels = None
    if not subtree:
        kstate = state
        kstate, _ = st._advance(kstate)           # warm the eager path
        torch.cuda.synchronize()
        _lib.kernel_times()                        # clear
        lib.hps_ktimer_enable(1)
        for _ in range(kt_steps):
            kstate, _ = st._advance(kstate)
        lib.hps_ktimer_enable(0)
        kt = _lib.kernel_times()
        kernels = kernel_table(kt, kt_steps, tree, lib, st, k)

    # e2e: public API with host state in / host result out every step
    e2e_steps = args.e2e_steps or max(3, args.steps // 2)
    uh = torch.empty((k, tree.N) if k > 1 else (tree.N,), dtype=torch.float64).pin_memory()
    uh.copy_(state.u_device.cpu())
    out = torch.empty_like(uh).pin_memory()
    t_e2e = state.t
    if subtree:   # the sharded stepper: synchronous public step with host state
        def e2e_step(src=uh, dst=out):
            s = st.step(hb.StepperState(t_e2e, src))
            dst.copy_(s.u_device, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            return ev
    else:         # step_host: every step copies its input in and its result out;
        def e2e_step(src=uh, dst=out):   # the copies of neighbouring (independent) steps overlap
            return st.step_host(t_e2e, src, dst)
    e2e_step()              # warm
    if not subtree:
        st.sync_host()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    last = None
    for _ in range(e2e_steps):
        last = e2e_step()
    torch.cuda.current_stream().wait_event(last)
    e1.record()
    if not subtree:
        st.sync_host()
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1))
    e2e_val = tree.N * 5 * e2e_steps * copies / (e2e_ms * 1e-3)
    nbytes = uh.numel() * 8
    # dependent trajectory: each step starts from the previous step's host result
    dep = None
    if not subtree:
        bufs = [uh, out]
        barrier()
        t0w = time.perf_counter()
        for i in range(e2e_steps):
            ev = st.step_host(t_e2e, bufs[i & 1], bufs[(i + 1) & 1])
            ev.synchronize()
        st.sync_host()
        dep_s = time.perf_counter() - t0w
        dep = {"value": tree.N * 5 * e2e_steps * copies / dep_s, "unit": UNIT,
               "ms_per_step": 1e3 * dep_s / e2e_steps, "clock": "host wall clock (each step waits for its result)"}

    # whole-solve roofline (plain solve): HBM bytes the layout requires vs FP64 work
    layout = st.ops.layout
    if layout == "shared":
        b_op, b_vec = solve_bytes_shared(tree, k)
    else:
        b_op, b_vec = solve_bytes(tree, k, prob.coeffs.is_constant)
    avg_solve = max_over_ranks(statistics.mean(solve_ms))
    if subtree:   # per-GPU share of the algorithmic bytes / flops (top levels counted once)
        b_op, b_vec = b_op / world, b_vec / world
    peak, src = peaks()
    flops = solve_flops(tree, k, tensor_leaf=getattr(st.ops, "leaf_solve", "dense") == "tensor")
    if subtree:
        flops /= world
    solve = {"solve_ms": avg_solve, "solves_timed": len(solve_ms), "layout": layout,
             "leaf_solve": getattr(st.ops, "leaf_solve", "dense"),
             "algorithmic_bytes_per_solve": b_op + b_vec, "gflops_per_solve": flops / 1e9,
             "frac_hbm": (b_op + b_vec) / (avg_solve * 1e-3) / (peak * 1e9),
             "frac_fp64": flops / (avg_solve * 1e-3) / (FP64_TFLOPS * 1e12),
             "traffic": profiled_traffic(f"{args.config}/{layout}")}

    # roofline: the dominant kernel of the step (largest share of the step time)
    top = max(kernels, key=lambda r: r["share_of_step"]) if kernels else None
    if top is not None and top.get("achieved_gbs"):
        traffic = profiled_kernel_traffic(args.config, top["kernel"])
        roof = {"bound": "hbm", "achieved": top["achieved_gbs"], "peak": peak, "unit": "GB/s",
                "peak_source": src, "frac": top["achieved_gbs"] / peak, "traffic": traffic,
                "kernel": top["kernel"], "us_per_launch": top["us_per_launch"],
                "algorithmic_bytes_per_launch": top["bytes_per_launch"],
                "share_of_step": top["share_of_step"]}
    else:   # no byte model for the dominant kernel (sharded solve, multi-rhs GEMMs): the whole stage solve
        t_hbm = (b_op + b_vec) / (peak * 1e9)
        t_fp64 = flops / (FP64_TFLOPS * 1e12)
        if t_hbm >= t_fp64:
            roof = {"bound": "hbm", "achieved": (b_op + b_vec) / (avg_solve * 1e-3) / 1e9, "peak": peak,
                    "unit": "GB/s", "peak_source": src}
        else:
            roof = {"bound": "tensor", "achieved": flops / (avg_solve * 1e-3) / 1e12, "peak": FP64_TFLOPS,
                    "unit": "TFLOP/s", "peak_source": "measured FP64 DMMA (profiles/r01_fp64_peak.txt)"}
        roof["frac"] = roof["achieved"] / roof["peak"]
        roof.update({"traffic": solve["traffic"], "kernel": "stage solve (hps_solve%s)" % ("_phase" if subtree else ""),
                     "dominant_kernel": None if top is None else top["kernel"]})

    # the bench's own 64x64 sample: one GPU step against the CPU oracle's step
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        val, sample, _, ostate = cpu_oracle_sample(cfg, 1, 0, keep_state=True)
        cpu = {"value": val, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
               "sample": sample}
        n_s = min(SAMPLE_N, cfg["n"])
        c_s = dict(cfg, n=n_s)
        tree_s = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), n_s, n_s, cfg["p"])
        st_s = hb.TimeStepper(tree_s, hb.ParabolicProblem(**make_problem(hb, c_s)), "ARK4", dt=cfg["dt"],
                              layout=args.layout)
        u_s = st_s.step(st_s.initial_state()).u
        parity["sample"] = f"{n_s}x{n_s} leaves, p={cfg['p']}, one ARK4 step vs the CPU oracle"
        parity["sample_rel_l2"] = float(np.linalg.norm(u_s - ostate) / np.linalg.norm(ostate))
    if parity:
        vals = [v for key, v in parity.items() if key in ("sample_rel_l2",)]
        parity["tolerance"] = 1e-10
        parity["ok"] = all(v <= 1e-10 for v in vals) and parity.get("manufactured_max_rel", 0.0) <= 1e-8

    if rank != 0:
        if distributed:
            dist.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (manufactured / seeded analytic fields; no dataset)",
        "config": config_block(cfg),
        "parallelism": (f"ensemble members sharded over {world} GPU(s)" if ensemble
                        else f"subtree-sharded over {world} GPUs (level-{world.bit_length() - 1} "
                             f"subtrees, NCCL flux all-gather per stage solve)" if subtree
                        else f"replicas x{world}"),
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": nbytes,
                "d2h_bytes_per_step": nbytes},
        "e2e_dependent": dep,
        "gpu_launches": int(launches),
        "roofline": roof,
        "kernels": kernels,
        "solve": solve,
        "parity": parity or None,
        "clocks": clk.summary(),
        "build_s": build_s,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if distributed:
        dist.destroy_process_group()


def profiled_kernel_traffic(config, kernel):
    """ncu dram bytes (read + write) per launch of ``kernel`` from the
    committed capture summary, if any (profiles/traffic_kernels.json)."""
    path = os.path.join(ROOT, "profiles", "traffic_kernels.json")
    try:
        with open(path) as fh:
            d = json.load(fh).get(config, {})
    except (OSError, ValueError):
        return None
    norm = lambda n: n.replace("true", "1").replace("false", "0").replace(" ", "")
    for name, v in d.items():
        if norm(name) == norm(kernel):
            return v
    return None


def kernel_table(kt, nsteps, tree, lib, st, k):
    """Per-kernel rows {kernel, launches_per_step, us_per_launch,
    share_of_step, bytes_per_launch, achieved_gbs, frac} from the event
    timings of ``nsteps`` eager steps (kernel_bytes gives the algorithmic
    bytes; None for kernels without a byte model)."""
    peak, _ = peaks()
    shapes = [(lm.count, lm.n3, lm.n12) for lm in tree.level_maps]
    dF = lib.hps_plan_fused_level(st.ops.plan.handle)
    nbd = tree.boundary_ids.size
    kb = kernel_bytes(shapes, dF, tree.L, tree.ni, tree.nb, nbd, tree.N, k,
                      per_node=getattr(st.ops, "layout", "shared") == "per_node")
    s = st.pair.s
    total = sum(v[0] for v in kt.values())
    # stage terms of the fused leaf-up kernel, stage i (1..s-1): u, L u_0..u_{i-1}, q's spatial parts
    nq = len(st._Q.sep) if st._Q.sep is not None else 0
    nqg = 1 if st.problem.g is not None else 0
    up_terms = [1 + i + nq + nqg * i for i in range(1, s)]
    rows = []
    for name, (tot_ms, cnt) in sorted(kt.items(), key=lambda kv: -kv[1][0]):
        per = tot_ms / cnt
        b = None
        if name.startswith("k_mega"):
            b = kb["k_mega"]
        elif name.startswith("k_sub_up"):
            b = kb["k_sub_up"]
        elif name.startswith("k_sub_down"):
            b = kb["k_sub_down"]
        elif name.startswith("k_leaf_fd_mma") and name.endswith(", 4>"):
            b = statistics.mean(kb["leaf_up_terms"](nt) for nt in up_terms)
        elif name.startswith("k_leaf_fd_mma") and name.endswith(", 2>"):
            b = kb["leaf_down"]
        elif name.startswith("k_leaf_fd_mma") and name.endswith(", 3>"):
            b = kb["leaf_lu"]
        elif name.startswith("k_root_dir"):
            b = kb["root_dir"](s - 1)
        row = {"kernel": name, "launches_per_step": cnt / nsteps, "us_per_launch": 1e3 * per,
               "share_of_step": tot_ms / total if total else None, "bytes_per_launch": b}
        if b:
            row["achieved_gbs"] = b / (per * 1e-3) / 1e9
            row["frac"] = row["achieved_gbs"] / peak
        rows.append(row)
    return rows


if __name__ == "__main__":
    main()
