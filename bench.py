"""Benchmark of the matrix-free tangent apply y = K(u_k) v on B200.

Contract: one JSON line on rank 0.
  * workload (the metric's config, BASELINE configs[2]): 64^3 Q4 hexahedra on
    the curved map x' = x + 0.1 sin(2 pi y) e_x (per-qp J0 stored), iNH
    (mu=1, kappa=1000), u0 amplitude 0.1 at pre-map coordinates with the
    scaled noise 1e-3*8/64 (the literal 1e-3 noise is inadmissible: the
    reference throws NonPositiveJacobian at (1, 46), reported under
    "workloads"), v seeded U[-1,1].  At N GPUs: weak scaling, one 64^3 z-slab
    per GPU (global mesh 64 x 64 x 64N), ghost faces exchanged with NCCL and
    overlapped with interior elements.
  * a "step" = one tangent apply of the headline variant (fp64, strategy
    none); the other cfg2 variants (fp64 tensor/scalar/cachedF, fp32
    none/tensor) are timed the same way under "variants"; cfg1 (32^3 Q3 cNH,
    12 variants) under "variants_cfg1" (N=1).
  * L2 is flushed (256 MiB write) before every timed apply (the cfg2 inputs
    are also larger than L2); each apply is timed with CUDA events on the
    operator's stream; max over ranks.
  * value = global DoFs / apply time (reference definition, runner.cpp:131-132).
  * e2e = the same metric through the public host-vector call
    (emfgpu_op_apply_host: pinned H2D of v, apply, D2H of y, sync).
  * --impl reference: the reference's own CPU implementation (oracle/_ref,
    ElasticOperator<double>, all host threads) on the same cfg2 workload,
    timed with runner.cpp:84-121's protocol (blocks of 1 apply, >= 1 s per
    measurement, average of the best 3).
"""
from __future__ import annotations

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

METRIC = "tangent-operator apply DoFs/s"
UNIT = "DoF/s"
# headline: BASELINE configs[2] (scaled-noise variant), per GPU
C2_N, C2_P, C2_MODEL = 64, 4, "inh"
C2_MU, C2_KAPPA, C2_SHEAR, C2_AMP = 1.0, 1000.0, 0.1, 0.1
C2_NOISE = 1e-3 * 8.0 / C2_N
# cfg1 sweep: BASELINE configs[1]
C1_N, C1_P = 32, 3
MU, LAM = 1.0, 10.0
P = C1_P

# Algorithmic work per element: reference sweep structure
# (8 forward + 9 transpose sweeps per component, u_k swept again when the
# strategy reads it) + counted qp flops of the reference material pipeline.
QP_FLOPS = {"cnh": {"none": 782, "scalar": 714, "tensor": 386, "cachedF": 746},
            "inh": {"none": 852, "scalar": 748, "tensor": 408, "cachedF": 816},
            "fiber": {"none": 1063, "scalar": 887, "tensor": 521, "cachedF": 1027}}
# ledger apply traffic per qp (paper_2408_12479_b200/ledger.py, the reference's
# ledger.cpp:22-76 restated and tested), with the u_k row removed (u_k counted
# per DoF) and, for the fibre model with one global frame, without the per-qp
# H4/H6 rows; cachedF (ours): J0 + G.
def ledger_qp_bytes(model, strategy, domain="material"):
    from paper_2408_12479_b200 import ledger as LG
    if strategy == "cachedF":
        return 144
    rows = [r for r in LG.cell_ledger(model, domain, strategy) if r[2] and r[0] not in ("u_k", "H4", "H6")]
    return sum(b for _, b, _ in rows)


def flops_per_element(strategy, n=P + 1, model="cnh"):
    reads_uk = strategy in ("none", "scalar")
    sf = (75 if reads_uk else 51) * n ** 3 * (2 * n - 1) + 9 * n ** 3
    return sf + n ** 3 * QP_FLOPS[model][strategy]


def bytes_per_apply(strategy, prec, ndofs, nel, n=P + 1, model="cnh"):
    """Algorithmic bytes (SURVEY.md §8(d) ledger minus the u_k row, u_k per DoF;
    geometry per qp is the yardstick even when stored per element)."""
    s = prec // 8
    nq = nel * n ** 3
    k = 3 if strategy in ("none", "scalar") else 2
    return ledger_qp_bytes(model, strategy) * s / 8 * nq + k * s * ndofs


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def read_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def nominal_fma_tflops(prec, sm_mhz=None, sms=148):
    """Nominal FMA-pipe peak: 64 FP64 / 128 FP32 FMA lanes per SM per clock
    (2 flops each) at the maximum SM clock."""
    mhz = sm_mhz or read_peaks().get("sm_max_mhz", 1965.0)
    return sms * (64 if prec == 64 else 128) * 2 * mhz * 1e6 / 1e12


def headline_config(world):
    """The config dict of the headline line, identical in both arms."""
    return {"workload": "cfg2 (BASELINE configs[2], scaled-noise variant): 64^3 Q4 per GPU, curved map "
                        "x'=x+0.1 sin(2 pi y) e_x with per-qp J0, iNH mu=1 kappa=1000, u0 amp 0.1 at pre-map "
                        "coords + noise 1e-3*8/64, v U[-1,1]; fp64, strategy none",
            "global_mesh": [C2_N, C2_N, C2_N * world], "degree": C2_P, "ndofs": 3 * (C2_N * C2_P + 1) ** 2 * (
                C2_N * world * C2_P + 1),
            "l2": "flushed (256 MiB write) before every timed apply; inputs (x 407 MB) exceed L2",
            "parallelism": f"z-slab x{world}"}


def c2_material(G):
    return G.MaterialParams(mu=C2_MU, lam=LAM, kappa_b=C2_KAPPA)


def c2_inputs(part):
    from paper_2408_12479_b200 import inputs as I
    u0 = I.make_u0_planes(part.nx, part.ny, part.nz, part.p, part.c0, part.c1, amp=C2_AMP, noise=C2_NOISE,
                          faces=part.faces, extent=(1.0, 1.0, float(part.world)))
    v = I.make_v_planes(part.nx, part.ny, part.nz, part.p, part.c0, part.c1)
    return u0, v


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# the reference's CPU path (oracle/_ref = the unmodified reference, built from
# its sources by oracle/Makefile)
def ref_cfg2_operator(threads, precision=64):
    """ElasticOperator<double> of the reference on the cfg2 level: build_cube
    lattice + the shear map, J0 recomputed by the reference's own sweeps
    (SURVEY §8(c) gap 1), linearized at the same seeded u0."""
    from oracle import refbind as R
    from paper_2408_12479_b200 import workloads as W
    L0 = R.RefLevel(1, 6, C2_P, 0.0, 1)
    c = L0.coords().reshape(-1, 3)
    c[:, 0] += C2_SHEAR * np.sin(2.0 * np.pi * c[:, 1])
    del L0
    L = R.RefLevel(1, 6, C2_P, 0.0, 1, coords=c.reshape(-1))
    del c
    w = W.cfg2()
    op = R.RefOperator(L, C2_MODEL, R.material_params(mu=C2_MU, lam=LAM, kappa=C2_KAPPA), "none", precision,
                       threads=threads)
    t0 = time.perf_counter()
    op.update_linearization(w.u0())
    t_lin = time.perf_counter() - t0
    return L, op, w.v(), t_lin


def runner_protocol(fn, measurements, min_seconds=1.0, average_best=3):
    """runner.cpp:84-121: after one warm-up call (done by the caller), each
    measurement repeats blocks of `fn` until min_seconds have passed (blocks
    of 1 apply: repetitions_block=1, SURVEY §8(d) for cfg2-4); the best
    `average_best` measurements (by rate) are averaged."""
    runs = []
    for _ in range(measurements):
        reps, t0 = 0, time.perf_counter()
        el = 0.0
        while el < min_seconds:
            fn()
            reps += 1
            el = time.perf_counter() - t0
        runs.append((reps, el))
    runs.sort(key=lambda r: -r[0] / r[1])
    keep = runs[:min(average_best, len(runs))]
    reps = sum(r for r, _ in keep)
    secs = sum(s for _, s in keep)
    return reps, secs, runs


def run_reference(args):
    """--impl reference: the reference's CPU ElasticOperator<double>
    (oracle/_ref), same cfg2 workload and config, all host threads,
    runner.cpp's protocol with blocks of 1 apply."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import refbind as R
    threads = os.cpu_count() or 1
    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libemfref.so not built"}))
        return
    L, op, v, t_lin = ref_cfg2_operator(threads)
    for _ in range(max(1, min(args.warmup, 1))):
        op.apply(v)
    meas = max(3, min(args.steps, 10))
    reps, secs, runs = runner_protocol(lambda: op.apply(v), meas)
    val = L.ndofs * reps / secs
    dt = secs / reps
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded splitmix64, SURVEY §8(c))",
        "config": headline_config(world),
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{meas} measurements of >=1 s of full cfg2 applies (64^3 Q4, {L.ndofs} DoFs; "
                                   f"the reference's HexMesh is one cube, so at N>1 this is the per-GPU slab "
                                   f"shape), best 3 averaged (runner.cpp:84-121, blocks of 1)"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference": {"update_linearization_s": t_lin, "threads": threads,
                      "runs": [[r, s] for r, s in runs]},
    }))


def cpu_baseline_sample(seconds=10.0):
    """Reference CPU path on the GPU box's host (rank 0, N=1): a bounded sample
    of the same cfg2 workload (oracle/_ref, all threads; the C port if the
    reference is not built)."""
    threads = os.cpu_count() or 1
    try:
        from oracle import refbind as R
        if not R.available():
            raise OSError
        L, op, v, t_lin = ref_cfg2_operator(threads)
        n = L.ndofs
        kind = "reference"
    except OSError:
        from oracle import orcbind as O
        from paper_2408_12479_b200 import workloads as W
        from paper_2408_12479_b200 import inputs as I
        w = W.cfg2()
        X, Y, Z = I.lattice_positions(C2_N, C2_N, C2_N, C2_P)
        X = X + C2_SHEAR * np.sin(2.0 * np.pi * Y)
        coords = np.stack([X, Y, Z], 1).ravel()
        op = O.OracleOperator(C2_N, C2_N, C2_N, C2_P, coords, 1, "inh",
                              np.array([C2_MU, LAM, C2_KAPPA, 2, 5, 3.62, 34.3, 0.7, 1, 0, 0, 0, 1, 0, 0, 0, 1]))
        t0 = time.perf_counter()
        op.update_linearization(w.u0())
        t_lin = time.perf_counter() - t0
        v = w.v()
        n = v.size
        kind = "port"
        threads = 1
    op.apply(v)
    k, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds or k < 2:
        op.apply(v)
        k += 1
    dt = (time.perf_counter() - t0) / k
    return {"value": n / dt, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{k} full cfg2 applies (64^3 Q4 iNH, {n} DoFs, ElasticOperator<double>, none, "
                      f"{threads} threads), {dt * 1e3:.0f} ms each; update_linearization {t_lin:.1f} s (serial)"}


# ---------------------------------------------------------------------------
def time_variant(G, args, lev, part, sop_cls, u0, v, model, params, prec, strat, flush, world, dist, ev_elem=True,
                 keep=False):
    """Times one operator variant: `steps` whole applies (L2 flushed before
    each, CUDA events on the stream), then the element kernel alone (N=1)."""
    import torch
    spatial = strat.startswith("spatial_")
    op = G.ElasticOperator(lev, model, params, strat.replace("spatial_", ""), prec,
                           domain="spatial" if spatial else "material")
    op.update_linearization(u0)
    dt = torch.float64 if prec == 64 else torch.float32
    sop = sop_cls(op, part, dt)
    x = torch.tensor(v, dtype=dt, device="cuda")
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        sop.apply(x, y)
    barrier()
    tot = []
    for _ in range(args.steps):
        flush.fill_(1.0)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(stream)
        # one GPU: the whole apply in one call (element kernel + node kernel
        # as its programmatic dependent); the element kernel is timed alone below
        sop.apply(x, y)
        ev[1].record(stream)
        ev[2].record(stream)
        tot.append(ev)
    barrier()
    ms = [e[0].elapsed_time(e[2]) for e in tot]
    if world == 1 and ev_elem:
        el = []
        for _ in range(args.steps):
            flush.fill_(1.0)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record(stream)
            op.apply_elements(x, 0, part.nz_local)
            ev[1].record(stream)
            el.append(ev)
        barrier()
        ms_el = [e[0].elapsed_time(e[1]) for e in el]
    else:
        ms_el = [e[0].elapsed_time(e[1]) for e in tot]
    t = torch.tensor([sum(ms) / len(ms), sum(ms_el) / len(ms_el), min(ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step, ms_elem, ms_min = t.tolist()
    rec = {"dofs_per_s": part.global_dofs / (ms_step * 1e-3), "ms_per_apply": ms_step, "ms_min": ms_min,
           "ms_element_kernel": ms_elem}
    kept = (op, sop, x, y) if keep else None
    if not keep:
        del op, sop, x, y
    return rec, kept


def add_roofline(rec, strat, prec, nel, ndofs, n, model, peaks):
    """Per-variant roofline fields of the element kernel: algorithmic flops
     against the nominal and the measured FMA peaks, ledger
    bytes against the measured HBM copy bandwidth."""
    t = rec["ms_element_kernel"] * 1e-3
    st = strat.replace("spatial_", "")
    if not strat.startswith("spatial_"):
        fl = flops_per_element(st, n, model) * nel
        rec["element_kernel_tflops"] = fl / t / 1e12
        rec["fma_frac_nominal"] = rec["element_kernel_tflops"] / peaks[f"nominal{prec}"]
        rec["fma_frac_measured"] = rec["element_kernel_tflops"] / peaks[f"measured{prec}"]
        by = bytes_per_apply(st, prec, ndofs, nel, n, model)
    else:
        k = 3 if st in ("none", "scalar") else 2
        by = ledger_qp_bytes(model, st, "spatial") * (prec // 8) / 8 * nel * n ** 3 + k * (prec // 8) * ndofs
    rec["element_kernel_gbs"] = by / t / 1e9
    rec["hbm_frac_yardstick"] = rec["element_kernel_gbs"] / peaks["hbm"]
    return rec


def add_real_traffic(rec, tr, hbm):
    """Beside the ledger yardstick: the DRAM bytes one launch of this variant
    really moves (profiles/traffic.json, from an ncu capture) over this run's
    element-kernel time, as a fraction of the measured HBM bandwidth."""
    if not tr:
        return rec
    rec["dram_bytes_per_launch_ncu"] = tr["dram_bytes_per_launch"]
    rec["hbm_frac_real_traffic"] = tr["dram_bytes_per_launch"] / (rec["ms_element_kernel"] * 1e-3) / 1e9 / hbm
    return rec


def load_traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def run_gpu(args):
    import torch
    import torch.distributed as dist
    from paper_2408_12479_b200 import emfgpu as G
    from paper_2408_12479_b200.slab import SlabPartition, SlabOperator

    world, rank, local = dist_env()
    world = max(world, 1)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    part = SlabPartition(C2_N, C2_N, C2_N * world, C2_P, world, rank, faces=1)
    params = c2_material(G)
    u0, v = c2_inputs(part)
    lev = part.make_level(extent=(1.0, 1.0, float(world)), device=local, map="shear_x", map_param=(C2_SHEAR,))
    flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
    peaks_file = read_peaks()
    hbm = peaks_file.get("hbm_gbs", 6650.0)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.__enter__()
    variants = {}
    rec, kept = time_variant(G, args, lev, part, SlabOperator, u0, v, C2_MODEL, params, 64, "none", flush, world,
                             dist, keep=True)
    if sampler:
        sampler.__exit__()
    variants["fp64_none"] = rec
    op, sop, x, y = kept
    launches = sop.launches_per_apply * args.steps

    # e2e through the public host-vector API (pinned host buffers)
    hx = torch.tensor(v, dtype=torch.float64).pin_memory()
    hy = torch.empty_like(hx).pin_memory()
    if world == 1:
        for _ in range(max(1, args.warmup)):
            G.lib().emfgpu_op_apply_host(op.h, hx.data_ptr(), hy.data_ptr())
        ts = []
        for _ in range(args.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            st = G.lib().emfgpu_op_apply_host(op.h, hx.data_ptr(), hy.data_ptr())
            ts.append(time.perf_counter() - t0)
            assert st == 0
        e2e_ms = 1e3 * sum(ts) / len(ts)
        call = "emfgpu_op_apply_host (pinned host vectors; H2D, apply, D2H pipelined in z-chunks)"
    else:
        ts = []
        dx = torch.empty_like(x)
        for _ in range(args.steps):
            barrier()
            t0 = time.perf_counter()
            dx.copy_(hx, non_blocking=True)
            sop.apply(dx, y)
            hy.copy_(y, non_blocking=True)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        tt = torch.tensor([sum(ts) / len(ts)], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = tt.item() * 1e3
        call = "SlabOperator.apply with pinned H2D/D2H per rank"
    e2e = {"value": part.global_dofs / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": hx.numel() * 8,
           "d2h_bytes_per_step": hy.numel() * 8, "ms_per_step": e2e_ms, "call": call}
    # evaluate_residual on the same operator (runner.cpp:85-105 times it too)
    res_rec = None
    if world == 1:
        du = torch.tensor(u0, dtype=torch.float64, device="cuda")
        r = torch.empty_like(du)
        for _ in range(2):
            op.evaluate_residual_device(du, r)
        torch.cuda.synchronize()
        evs = []
        for _ in range(max(3, args.steps // 2)):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            op.evaluate_residual_device(du, r)
            e1.record()
            evs.append((e0, e1))
        torch.cuda.synchronize()
        ms_r = sum(a.elapsed_time(b) for a, b in evs) / len(evs)
        res_rec = {"dofs_per_s": lev.n_dofs / (ms_r * 1e-3), "ms": ms_r, "strategy": "none (fp64)"}
        del du, r
    del op, sop, x, y, kept

    for prec, strat in ((64, "tensor"), (64, "scalar"), (64, "cachedF"), (32, "none"), (32, "tensor"),
                        (32, "cachedF"), (32, "scalar")):
        rec, _ = time_variant(G, args, lev, part, SlabOperator, u0, v, C2_MODEL, params, prec, strat, flush, world,
                              dist)
        variants[f"fp{prec}_{strat}"] = rec

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    fp64_meas = G.fma_peak_tflops(64, 0.5)
    fp32_meas = G.fma_peak_tflops(32, 0.5)
    clocks = sampler.summary() if sampler else None
    peaks = {"nominal64": nominal_fma_tflops(64), "nominal32": nominal_fma_tflops(32), "measured64": fp64_meas,
             "measured32": fp32_meas, "hbm": hbm}
    traffic = load_traffic()
    for k, r in variants.items():
        prec, strat = (64 if k.startswith("fp64") else 32), k.split("_", 1)[1]
        add_roofline(r, strat, prec, part.nel_local, lev.n_dofs, C2_P + 1, C2_MODEL, peaks)
        add_real_traffic(r, traffic.get("cfg2_" + k), hbm)
    head = variants["fp64_none"]
    tr = traffic.get("cfg2_fp64_none")
    fl = flops_per_element("none", C2_P + 1, C2_MODEL) * part.nel_local
    line = {
        "metric": METRIC, "value": head["dofs_per_s"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms_per_apply"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: seeded splitmix64 u0/v (SURVEY §8(c)), mesh and J0 generated for each slab",
        "config": headline_config(world),
        "roofline": {"bound": "fp64_fma", "achieved": head["element_kernel_tflops"], "peak": peaks["nominal64"],
                     "unit": "TFLOP/s", "frac": head["element_kernel_tflops"] / peaks["nominal64"],
                     "traffic": tr["dram_bytes_per_launch"] if tr else None,
                     "kernel": "apply_v2_kernel<double,4,INH,S_NONE,curved> (element phase)",
                     "peak_source": "nominal FP64: 148 SMs x 64 FMA/clk x 2 x sm_max_mhz (MEASURED_PEAKS.json "
                                    "has no FP64 entry)",
                     "peak_measured_fma_loop": fp64_meas,
                     "frac_of_measured_fma_loop": head["element_kernel_tflops"] / fp64_meas,
                     "flops_per_launch": fl, "flops_per_element": flops_per_element("none", C2_P + 1, C2_MODEL),
                     "elements_per_launch": part.nel_local,
                     "hbm_achieved_gbs_yardstick": head["element_kernel_gbs"], "hbm_peak_gbs": hbm,
                     "traffic_source": tr.get("source") if tr else None,
                     "traffic_frac_of_hbm": (tr["dram_bytes_per_launch"] / (head["ms_element_kernel"] * 1e-3) / 1e9
                                             / hbm) if tr else None},
        "fma_peaks_tflops": {"fp64_nominal": peaks["nominal64"], "fp32_nominal": peaks["nominal32"],
                             "fp64_measured_fma_loop": fp64_meas, "fp32_measured_fma_loop": fp32_meas},
        "variants": variants,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if res_rec:
        line["residual"] = res_rec
    if world == 1 and not args.no_extra:
        line["variants_cfg1"] = run_cfg1_sweep(args, flush, peaks)
        for k, r in line["variants_cfg1"].items():
            add_real_traffic(r, traffic.get("cfg1_" + k), hbm)
        line["workloads"] = run_extra_workloads(args, flush, peaks)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample(args.cpu_seconds)
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def run_cfg1_sweep(args, flush, peaks):
    """BASELINE configs[1] (32^3 affine cube Q3 cNH): fp64/fp32 x
    none/cachedF/scalar/tensor + the spatial domain, one GPU."""
    from paper_2408_12479_b200 import emfgpu as G
    from paper_2408_12479_b200 import inputs as I
    from paper_2408_12479_b200.slab import SlabPartition, SlabOperator
    part = SlabPartition(C1_N, C1_N, C1_N, C1_P, 1, 0, faces=1)
    lev = part.make_level()
    u0 = I.make_u0(C1_N, C1_N, C1_N, C1_P)
    v = I.make_v(u0.size)
    params = G.MaterialParams(mu=MU, lam=LAM)
    out = {}
    order = [(64, "none"), (64, "cachedF"), (64, "scalar"), (64, "tensor"),
             (32, "none"), (32, "cachedF"), (32, "scalar"), (32, "tensor"),
             (64, "spatial_none"), (64, "spatial_tensor"), (32, "spatial_none"), (32, "spatial_tensor")]
    for prec, strat in order:
        rec, _ = time_variant(G, args, lev, part, SlabOperator, u0, v, "cnh", params, prec, strat, flush, 1, None)
        out[f"fp{prec}_{strat}"] = add_roofline(rec, strat, prec, part.nel_local, lev.n_dofs, C1_P + 1, "cnh",
                                                peaks)
    return out


def run_extra_workloads(args, flush, peaks):
    """BASELINE configs 3 and 4 on one GPU (variants documented in
    paper_2408_12479_b200/workloads.py), and the literal cfg2/cfg4 inputs'
    rejection points."""
    import torch
    from paper_2408_12479_b200 import emfgpu as G
    from paper_2408_12479_b200 import workloads as W
    out = {}
    # cfg4 (well-posed variant): fp64 PCG + fp32 hp-MG V-cycle
    w = W.cfg4(wellposed=True)
    lev = w.level()
    t0 = time.perf_counter()
    op = G.ElasticOperator(lev, w.model, w.material(), "none", 64)
    u0 = np.zeros(lev.n_dofs)
    op.update_linearization(u0)
    mg = G.MgHierarchy(lev, w.model, w.material(), degree=5, coarse_n=6, precision=32)
    mg.update_linearization(torch.zeros(lev.n_dofs, dtype=torch.float64, device="cuda"))
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    b = torch.tensor(W.rhs(w), device="cuda")
    x = torch.empty_like(b)
    # warm-up: two PCG iterations load every kernel of the solve (lazy module
    # loading) before the timed solve
    try:
        G.pcg_solve(op, mg, b, x, 1e-8, 2)
    except G.EmfGpuError:
        pass  # not converged in 2 iterations: expected
    torch.cuda.synchronize()
    smp = ClockSampler(torch.cuda.current_device())
    smp.__enter__()
    t0 = time.perf_counter()
    its, hist = G.pcg_solve(op, mg, b, x, 1e-8, 300)
    torch.cuda.synchronize()
    t_solve = time.perf_counter() - t0
    smp.__exit__()
    ref4 = None
    try:
        with open(os.path.join(ROOT, "tests", "golden", "cfg4_full.json")) as f:
            ref4 = json.load(f)
    except (OSError, ValueError):
        pass
    out["cfg4_wellposed"] = {"ndofs": lev.n_dofs, "levels": mg.levels(), "cg_iterations": its,
                             "final_rel_residual": float(hist[-1]), "solve_s": t_solve,
                             "ms_per_iteration": 1e3 * t_solve / max(its, 1), "setup_s": t_setup,
                             "clocks": smp.summary(),
                             "settings": "iNH kappa/mu=50, u0=0, affine 48^3 Q4; fp64 PCG rtol 1e-8; fp32 V-cycle "
                                         "Q4->Q2->Q1->24^3->12^3->6^3, Chebyshev-Jacobi degree 5, dense coarse "
                                         "solve (1029 DoFs < coarse_direct_limit 2000, as the reference)"}
    if ref4:
        out["cfg4_wellposed"].update({
            "reference_iterations_dense_lu": ref4["iterations"], "reference_solve_s": ref4["solve_s"],
            "reference_setup_s": ref4["setup_s"], "reference_threads": ref4["threads"],
            "reference_note": "the reference's MgHierarchy<float> + fp64 PCG (oracle/ref_driver.cpp "
                              "ref_pcg_solve) run once in the build container (tests/golden/cfg4_full.json); "
                              "its dense coarse LU mishandles row pivots (solver.hpp:55-78, DESIGN.md §5), "
                              "so its iteration count with the dense coarse solve is not the parity target"})
        out["cfg4_literal"] = ref4.get("literal")
    try:
        with open(os.path.join(ROOT, "tests", "golden", "cfg4_full_cg.json")) as f:
            ref4cg = json.load(f)
        out["cfg4_wellposed"].update({"reference_iterations_cg_coarse": ref4cg["iterations"],
                                      "reference_cg_coarse_solve_s": ref4cg["solve_s"],
                                      "reference_cg_coarse_setup_s": ref4cg["setup_s"],
                                      "iterations_within_1_of_reference": abs(its - ref4cg["iterations"]) <= 1})
    except (OSError, ValueError):
        pass
    # the same solve with the V-cycle's level operators on strategy tensor
    # (the cached push-forward state: 19 fp32 fields per point instead of the
    # on-the-fly recomputation; the strategy is MgHierarchy's argument in the
    # reference too, solver.hpp:442)
    del mg, op
    t0 = time.perf_counter()
    op = G.ElasticOperator(lev, w.model, w.material(), "tensor", 64)  # the outer fp64 operator on tensor too
    op.update_linearization(u0)
    mgt = G.MgHierarchy(lev, w.model, w.material(), strategy="tensor", degree=5, coarse_n=6, precision=32)
    mgt.update_linearization(torch.zeros(lev.n_dofs, dtype=torch.float64, device="cuda"))
    torch.cuda.synchronize()
    t_setup_t = time.perf_counter() - t0
    try:
        G.pcg_solve(op, mgt, b, x, 1e-8, 2)
    except G.EmfGpuError:
        pass
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    its_t, hist_t = G.pcg_solve(op, mgt, b, x, 1e-8, 300)
    torch.cuda.synchronize()
    t_solve_t = time.perf_counter() - t0
    out["cfg4_wellposed"]["tensor_levels"] = {"cg_iterations": its_t, "final_rel_residual": float(hist_t[-1]),
                                              "solve_s": t_solve_t, "ms_per_iteration": 1e3 * t_solve_t / max(its_t, 1),
                                              "setup_s": t_setup_t,
                                              "settings": "outer fp64 operator and the fp32 V-cycle levels on strategy "
                                                          "tensor (cached push-forward state)"}
    del op, mgt, lev, b, x
    # cfg4 literal: rejected like the reference
    w = W.cfg4(wellposed=False)
    lev = w.level()
    op = G.ElasticOperator(lev, w.model, w.material(), "none", 64)
    try:
        op.update_linearization(w.u0())
        lit = {"admissible": True}
    except G.NonPositiveJacobian as ex:
        lit = {"admissible": False, "first_bad_element": ex.element, "first_bad_qpoint": ex.qpoint}
    out["cfg4_literal_gpu"] = lit
    del op, lev
    # cfg2 literal: rejected like the reference (first (e, q) = (1, 46))
    w = W.cfg2(literal=True)
    lev = w.level()
    op = G.ElasticOperator(lev, w.model, w.material(), "none", 64)
    try:
        op.update_linearization(w.u0())
        out["cfg2_literal"] = {"admissible": True}
    except G.NonPositiveJacobian as ex:
        out["cfg2_literal"] = {"admissible": False, "first_bad_element": ex.element, "first_bad_qpoint": ex.qpoint}
    del op, lev
    # cfg3: fibre tube with per-qp cylindrical frames, tensor strategy
    w = W.cfg3()
    lev = w.level()
    u0 = W.tube_u0(w, lev.node_coords())
    v = w.v()
    rec3 = {"mesh": "tube r=[1,1.3] L=10, 16x128x256 Q3, periodic theta, per-qp fibre frames",
            "ndofs": lev.n_dofs}
    for prec in (64, 32):
        op = G.ElasticOperator(lev, "fiber", w.material(), "tensor", prec)
        op.set_fibre_frame("cylindrical")
        op.update_linearization(u0)
        dt = torch.float64 if prec == 64 else torch.float32
        x = torch.tensor(v, dtype=dt, device="cuda")
        y = torch.empty_like(x)
        for _ in range(3):
            op.apply_tangent_device(x, y)
        ms = []
        for _ in range(max(3, args.steps // 4)):
            flush.fill_(1.0)
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record()
            op.apply_elements(x, 0, lev.nz)
            e1.record()
            op.apply_nodes(x, y, 0, lev.nz * lev.p)
            e2.record()
            ms.append((e0, e1, e2))
        torch.cuda.synchronize()
        t_all = sum(a.elapsed_time(c) for a, b, c in ms) / len(ms)
        t_el = sum(a.elapsed_time(b) for a, b, c in ms) / len(ms)
        nq = lev.n_elements * 64
        by = (ledger_qp_bytes("fiber", "tensor") + 96) * (prec // 8) / 8 * nq + 2 * (prec // 8) * lev.n_dofs
        rec3[f"fp{prec}_tensor"] = add_real_traffic(
            {"dofs_per_s": lev.n_dofs / (t_all * 1e-3), "ms_per_apply": t_all, "ms_element_kernel": t_el,
             "hbm_frac_yardstick": by / (t_el * 1e-3) / 1e9 / peaks["hbm"]},
            load_traffic().get(f"cfg3_fp{prec}_tensor"), peaks["hbm"])
        del op, x, y
    out["cfg3"] = rec3
    del lev
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-extra", action="store_true", help="skip the cfg1 sweep and the cfg3 / cfg4 workloads")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
