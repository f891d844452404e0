#!/usr/bin/env python
"""Benchmark of the joint psi/q CG iteration (arXiv 2407.20304 hot path) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg3] [--impl holo|reference]

One step = one Dai-Yuan CG iteration over the whole local shard (direction +
trial point + line-search sweep(s); every sweep = forward, amplitude residual,
both Wirtinger gradients, the grad_q / scalar allreduce and the DY dots).
Metric (BASELINE.json): frame-iterations/s = iterations/s x projections x distances,
whole job (all ranks).  Default workload: cfg3 (2048^2 projections on a 4096^2
torus, 4 distances) at 180 angles per GPU = the 8-GPU shard of the 1440-angle job
(weak scaling: 540 GiB of CG state needs 8 x B200).  Inputs are synthetic (synth/),
resident in HBM, each step touches >> L2 (126 MB).

For N > 1 launch with torchrun (one rank per GPU, NCCL).  --impl reference times the
fp64 oracle (test infrastructure, oracle/) on the host cores instead.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402

METRIC = "joint psi/q CG iters/s x projections x distances at 2048^2; % of HBM roofline"
UNIT = "frame-iterations/s"
FP32_LANES_PER_SM, N_SM = 128, 148


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        pk = json.load(open(path))
        return float(pk["hbm_gbs"]), float(pk.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return 6650.0, 1965.0, "fallback"


def fp32_peak(device):
    """P_FP32 measured by the in-repo FFMA microbenchmark (tools/fp32peak.cu), with the SM clock
    it ran at; falls back to the nominal 148 SM x 128 lanes x 2 x max clock if the tool is absent."""
    import ctypes
    lib = os.path.join(ROOT, "tools", "libfp32peak.so")
    try:
        if not os.path.exists(lib):
            import __graft_entry__
            __graft_entry__.build_tools()
        f = ctypes.CDLL(lib).fp32_peak
        f.argtypes = [ctypes.c_int, ctypes.c_double] + [ctypes.POINTER(ctypes.c_double)] * 3
        a, b, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        if f(device, 60.0, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)) == 0 and a.value > 0:
            return {"ffma_tflops": a.value, "ffma_fadd_tflops": b.value, "sm_mhz": c.value,
                    "source": "measured: tools/fp32peak.cu (FFMA chains, 148 x 8 CTAs x 256 threads)"}
    except Exception as e:  # pragma: no cover
        print(f"fp32 microbenchmark unavailable: {e}", file=sys.stderr)
    _, mhz, _ = peaks()
    return {"ffma_tflops": N_SM * FP32_LANES_PER_SM * 2 * mhz * 1e6 / 1e12, "ffma_fadd_tflops": None,
            "sm_mhz": mhz, "source": "nominal 148 SM x 128 lanes x 2 x max clock"}


# SURVEY 8(a) algorithmic HBM bytes per frame and pass, in units of A = 8 L^2 (N_z = 4 schedule;
# X1 counts the psi / eta / g state I/O of the CG step amortised over the planes).  B_min = sum.
ALG_BYTES_A = {"X1": 2.25, "Y1": 1.5, "X2": 1.125, "Y2": 2.5, "X3": 1.5}
B_MIN_A = 8.875


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def c_oracle_frames():
    """The naive-DFT C oracle (oracle/holo_oracle.c, OpenMP, fp64) timed per frame on all 8 frames
    of cfg0 and 8 frames (2 angles x 4 planes) of cfg1 -- SURVEY 8(d)'s oracle timing."""
    import oracle
    out = {}
    for name, K in (("cfg0", 4), ("cfg1", 2)):
        cfg = synth.CONFIGS[name]
        g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
        psi = synth.psi_stack(cfg, K=K).numpy()
        q = synth.probe(cfg).numpy()
        s = synth.shifts(cfg, K=K)
        d = np.abs(oracle.fwd(g, psi, q, s, cfg.n))
        t0 = time.perf_counter()
        oracle.grad(g, np.ones_like(psi), 0.9 * q, s, d)
        dt = time.perf_counter() - t0
        out[name] = {"frames": K * cfg.nz, "s_per_frame": dt / (K * cfg.nz),
                     "frame_it_per_s": K * cfg.nz / dt}
    return out


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        rows = [r for r in self.rows if len(r) >= 8]
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def workload(name, world, rank, angles):
    cfg = synth.CONFIGS[name]
    if angles:
        K = angles
        scaling = "weak"
    elif name == "cfg3":
        K, scaling = cfg.n_angles // 8, "weak"  # 180 per GPU: the 8-GPU shard of 1440 angles
    else:
        K, scaling = cfg.n_angles // world, "strong"
    return cfg, K, rank * K, scaling


def cpu_baseline(cfg, k=0, j=1):
    """Time the numpy/BLAS fp64 oracle (as it stands) on ONE frame (k, j) of the workload."""
    import oracle
    from oracle import np_oracle as npo
    try:
        from threadpoolctl import threadpool_info
        cores = max([t.get("num_threads", 0) for t in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    pr = npo.Problem(g, cfg.npad, cfg.n)
    psi_t = synth.psi_stack(cfg, K=1, k0=k).numpy()
    q_t = synth.probe(cfg).numpy()
    s = synth.shifts(cfg)[k:k + 1]
    qj = pr.qj(q_t, j)
    pr.mag(j)  # per-plane chirp-z matrix, built once per plane (oracle as it stands)
    w, _ = pr.frame_fwd(psi_t[0], qj, j, s[0, j])
    d = np.abs(w)
    t0 = time.perf_counter()
    pr.frame_grad(np.ones_like(psi_t[0]), qj, j, s[0, j], d)
    dt = time.perf_counter() - t0
    return {"value": 1.0 / dt, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"1 frame (k={k}, j={j}) of {cfg.name}: F + grad_psi + grad_q term on the "
                      f"{cfg.npad}^2 torus, numpy/BLAS fp64 oracle (oracle/np_oracle.py); {dt:.2f} s",
            "c_oracle_naive_dft": c_oracle_frames()}


def run_reference(args):
    """--impl reference: the fp64 oracle timed on the host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = synth.CONFIGS[args.workload]
    import oracle
    from oracle import np_oracle as npo
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    if cfg.name == "cfg4":
        return run_reference_ref_arm(args, cfg, g, npo)
    pr = npo.Problem(g, cfg.npad, cfg.n)
    K = 2
    psi_t = synth.psi_stack(cfg, K=K).numpy()
    q_t = synth.probe(cfg).numpy()
    s = synth.shifts(cfg)[:K]
    frames = [(k, j) for k in range(K) for j in range(cfg.nz)]
    qjs = {j: pr.qj(q_t, j) for j in range(cfg.nz)}
    data = {}
    for (k, j) in frames[: args.steps + args.warmup]:
        data[(k, j)] = np.abs(pr.frame_fwd(psi_t[k], qjs[j], j, s[k, j])[0])
    seq = [frames[i % len(frames)] for i in range(args.steps + args.warmup)]
    for (k, j) in seq[: args.warmup]:
        pr.frame_grad(np.ones_like(psi_t[k]), qjs[j], j, s[k, j], data.get((k, j), 1.0))
    t0 = time.perf_counter()
    for (k, j) in seq[args.warmup:]:
        pr.frame_grad(np.ones_like(psi_t[k]), qjs[j], j, s[k, j], data.get((k, j), 1.0))
    dt = time.perf_counter() - t0
    value = args.steps / dt
    try:
        from threadpoolctl import threadpool_info
        cores = max([t.get("num_threads", 0) for t in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    sample = (f"{args.steps} frames (one (k, j) frame per step, cycling over 2 angles x {cfg.nz} planes) of "
              f"{cfg.name}: F + grad_psi + grad_q term each, numpy/BLAS fp64 oracle")
    print(json.dumps({"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
                      "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
                      "impl": "reference", "dtype": "f64", "data": "synthetic",
                      "config": {"workload": cfg.name, "n": cfg.n, "npad": cfg.npad, "distances": cfg.nz},
                      "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                                       "sample": sample},
                      "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                      "vs_baseline": None}))


def setup_reference_arm(args, world, rank, local, dev, hb, JointCG):
    """configs[4]: probe-only retrieval from R = 64 x 4 reference frames (psi = 1, reading C16),
    q-only CG (rho_psi unused, no angles); frames sharded over ranks, grad_q allreduced."""
    cfg = synth.CONFIGS["cfg4"]
    R_total = cfg.n_angles
    R = R_total // world
    r0 = rank * R
    plan = hb.Plan(cfg.n, cfg.npad, cfg.z1, 0, cfg.wavelength, cfg.Z, cfg.det_pixel, device=local)
    plan.set_ref_shifts(synth.ref_shifts(cfg)[r0:r0 + R])
    q_t = synth.probe(cfg, device=dev, dtype=torch.complex64)
    w = torch.empty(R, cfg.n, cfg.n, dtype=torch.complex64, device=dev)
    plan.fwd_ref(q_t, w)
    inten = w.abs().square_()
    del w
    sqrt_dref = synth.poisson_amplitude(inten, cfg.photons, cfg, item=rank).float().contiguous()
    del inten
    torch.cuda.empty_cache()
    rho_q = args.rho_q if args.rho_q is not None else 1.0 / R_total
    q0 = (q_t * torch.exp(0.2j * torch.linspace(-1, 1, cfg.npad, device=dev))[None, :]).contiguous()
    solver = JointCG(plan, torch.zeros(0, device=dev), torch.ones(0, cfg.npad, cfg.npad, dtype=torch.complex64,
                                                                  device=dev), q0, rho_psi=0.0, rho_q=rho_q,
                     sqrt_dref=sqrt_dref)
    conf = {"workload": f"cfg4: probe-only, {R_total} reference frames of {cfg.n}^2 on a {cfg.npad}^2 torus "
                        f"(64 shifts x 4 distances), {R} per GPU", "frames_per_gpu": R, "frames_total": R_total,
            "n": cfg.n, "npad": cfg.npad, "rho_q": rho_q, "parallelism": f"frame-sharded dp{world}",
            "l2": "inputs > L2 (each step streams >= 10 GB per GPU; no flush needed)"}
    return plan, solver, R_total, conf, sqrt_dref, "strong", cfg


def cpu_baseline_ref(cfg):
    """The numpy fp64 O14 oracle on ONE reference frame of configs[4] (6144^2 torus)."""
    import oracle
    from oracle import np_oracle as npo
    try:
        from threadpoolctl import threadpool_info
        cores = max([t.get("num_threads", 0) for t in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    q = synth.probe(cfg).numpy()
    rs = synth.ref_shifts(cfg)[:1]
    d = np.ones((1, cfg.n, cfg.n))
    t0 = time.perf_counter()
    npo.grad_ref(g.wavelength, g.p0, g.zeta[0], q, rs, d)
    dt = time.perf_counter() - t0
    return {"value": 1.0 / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"1 reference frame of cfg4: F_ref + grad_q term on the {cfg.npad}^2 torus, numpy fp64 "
                      f"oracle (oracle/np_oracle.grad_ref); {dt:.2f} s"}


def run_reference_ref_arm(args, cfg, g, npo):
    """--impl reference for configs[4]: the numpy fp64 O14 oracle, one reference frame per step."""
    q = synth.probe(cfg).numpy()
    rs = synth.ref_shifts(cfg)
    d = np.ones((1, cfg.n, cfg.n))
    for i in range(args.warmup):
        npo.grad_ref(g.wavelength, g.p0, g.zeta[0], q, rs[i:i + 1], d)
    t0 = time.perf_counter()
    for i in range(args.steps):
        npo.grad_ref(g.wavelength, g.p0, g.zeta[0], q, rs[i:i + 1], d)
    dt = time.perf_counter() - t0
    value = args.steps / dt
    try:
        from threadpoolctl import threadpool_info
        cores = max([t.get("num_threads", 0) for t in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    sample = f"{args.steps} reference frames (one per step) of cfg4: F_ref + grad_q term, numpy fp64 oracle"
    print(json.dumps({"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
                      "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
                      "impl": "reference", "dtype": "f64", "data": "synthetic",
                      "config": {"workload": cfg.name, "n": cfg.n, "npad": cfg.npad},
                      "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                                       "sample": sample},
                      "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                      "vs_baseline": None}))


def run_multires(args, cfg, hb, dev, local, k0):
    """3-level schedule [(4, it), (2, it), (1, it)] through multires.run_schedule on K angles of the
    workload: data = |holo_fwd(truth)| + Poisson at full resolution, binned on the GPU per level;
    initial guess psi = 1, q = 0.9 x the 4x4 block mean of the true probe.  Per-level CUDA-event times."""
    from paper_2407_20304_b200 import multires
    K, it = args.multires_angles, args.multires_iters
    plan = hb.Plan(cfg.n, cfg.npad, cfg.z1, K, cfg.wavelength, cfg.Z, cfg.det_pixel, device=local,
                   angle_batch=min(args.batch, K))
    s = synth.shifts(cfg)[k0:k0 + K]
    plan.set_shifts(s)
    q_t = synth.probe(cfg, device=dev, dtype=torch.complex64)
    psi_t = synth.psi_stack(cfg, K=K, device=dev, dtype=torch.complex64, k0=k0)
    w = torch.empty(K, cfg.nz, cfg.n, cfg.n, dtype=torch.complex64, device=dev)
    plan.fwd(psi_t, q_t, w)
    sqrt_d = synth.poisson_amplitude(w.abs().square_(), cfg.photons, cfg, item=99).float().contiguous()
    del w, psi_t, plan
    f0 = 4
    Lc = cfg.npad // f0
    q0 = (0.9 * q_t.reshape(Lc, f0, Lc, f0).mean(dim=(1, 3))).contiguous()
    psi0 = torch.ones(K, Lc, Lc, dtype=torch.complex64, device=dev)
    levels = [(4, it), (2, it), (1, it)]
    marks = []

    def on_level(h):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks.append((h, e))

    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record()
    multires.run_schedule(levels, sqrt_d, s, cfg.n, cfg.npad, cfg.z1, cfg.wavelength, cfg.Z, cfg.det_pixel, psi0, q0,
                          rho_q=1.0 / K, device=local, angle_batch=min(args.batch, K), on_level=on_level)
    torch.cuda.synchronize()
    out, prev = [], e0
    for (h, e) in marks:
        ms = prev.elapsed_time(e)
        f = h["factor"]
        frames = K * cfg.nz * h["iterations"]
        out.append({"factor": f, "npad": cfg.npad // f, "n": cfg.n // f, "iterations": h["iterations"],
                    "sweeps": h["sweeps"], "F_start": h["F_start"], "F_end": h["F_end"], "ms": ms,
                    "frame_it_per_s": frames / (ms / 1e3)})
        prev = e
    return {"angles": K, "levels": out, "total_ms": e0.elapsed_time(prev),
            "note": "each level's ms includes its plan creation, data binning, upsampling and CG iterations"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--angles", type=int, default=0, help="angles per GPU (default: workload shard)")
    ap.add_argument("--impl", default="holo", choices=["holo", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--rho-q", type=float, default=None)
    ap.add_argument("--batch", type=int, default=8, help="angle_batch of the plan (angles per Y1/X2/Y2 launch; 16 is 1 % faster at 32 angles but does not fit 180 angles in 178 GiB next to the CG state)")
    ap.add_argument("--multires-angles", type=int, default=16,
                    help="angles of the timed 3-level multiresolution run (SURVEY 8(f) row 3); 0 = skip")
    ap.add_argument("--multires-iters", type=int, default=3, help="CG iterations per level of that run")
    ap.add_argument("--probe-shifts", type=float, default=0.0,
                    help="per-frame probe shifts s^p ~ U[-S, S] px (SURVEY 8(f) row 1, holo_set_probe_shifts); 0 = off")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2407_20304_b200 as hb
    from paper_2407_20304_b200.solver import JointCG

    dev = torch.device("cuda", local)
    if args.workload == "cfg4":
        plan, solver, frames, conf, sqrt_d, scaling, cfg = setup_reference_arm(args, world, rank, local, dev, hb,
                                                                              JointCG)
        K_total = 0
    else:
        cfg, K, k0, scaling = workload(args.workload, world, rank, args.angles)
        plan = hb.Plan(cfg.n, cfg.npad, cfg.z1, K, cfg.wavelength, cfg.Z, cfg.det_pixel, device=local,
                       angle_batch=min(args.batch, K))
        plan.set_shifts(synth.shifts(cfg)[k0:k0 + K] if k0 + K <= cfg.n_angles else
                        np.resize(synth.shifts(cfg), (k0 + K, cfg.nz, 2))[k0:k0 + K])
        if args.probe_shifts > 0:  # the f-1 path: q_kj = P_omega S_{s^p_kj} q in the data and in every sweep
            sp = np.random.default_rng([240720304, 7, rank]).uniform(-args.probe_shifts, args.probe_shifts,
                                                                    size=(K, cfg.nz, 2))
            plan.set_probe_shifts(sp)
        # ---- synthetic measurement: |forward(truth)|^2 with Poisson noise (bench input, not a parity value)
        q_t = synth.probe(cfg, device=dev, dtype=torch.complex64)
        psi_t = synth.psi_stack(cfg, K=K, device=dev, dtype=torch.complex64, k0=k0)
        w = torch.empty(K, cfg.nz, cfg.n, cfg.n, dtype=torch.complex64, device=dev)
        plan.fwd(psi_t, q_t, w)
        del psi_t
        inten = w.abs().square_()
        del w
        sqrt_d = synth.poisson_amplitude(inten, cfg.photons, cfg, item=rank).float().contiguous()
        del inten
        torch.cuda.empty_cache()
        K_total = K * world
        rho_q = args.rho_q if args.rho_q is not None else 1.0 / (K_total)
        solver = JointCG(plan, sqrt_d, torch.ones(K, cfg.npad, cfg.npad, dtype=torch.complex64, device=dev),
                         (0.9 * q_t).contiguous(), rho_psi=1.0, rho_q=rho_q)
        del q_t
        frames = K_total * cfg.nz
        conf = {"workload": f"{cfg.name}: {cfg.n}^2 projections on a {cfg.npad}^2 torus, {cfg.nz} distances, "
                            f"{K} angles per GPU ({K_total} total)",
                "angles_per_gpu": K, "angles_total": K_total, "distances": cfg.nz, "n": cfg.n,
                "npad": cfg.npad, "rho_q": rho_q, "angle_batch": plan.angle_batch,
                "parallelism": f"angle-sharded dp{world}",
                "probe_shifts": args.probe_shifts or None,
                "l2": "inputs > L2 (each step streams >= 25 GB per GPU; no flush needed)"}
    solver.start()
    for _ in range(args.warmup):
        solver.iterate()
    # ---- timed region
    sampler = ClockSampler(local)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler.start()
    time.sleep(0.3)
    l0, sw0 = plan.launch_count, solver.sweeps
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    hist = [solver.iterate() for _ in range(args.steps)]
    ev1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1)
    launches = plan.launch_count - l0
    sweeps = solver.sweeps - sw0
    # ---- per-pass CUDA events on the plan's stream: a SEPARATE run of the same steps, so the
    #      event records do not perturb the timed region above
    plan.profile_read(reset=True)
    plan.profile_enable(True)
    pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pe0.record()
    for _ in range(args.steps):
        solver.iterate()
    pe1.record()
    torch.cuda.synchronize()
    plan.profile_enable(False)
    ms_prof = pe0.elapsed_time(pe1)
    prof = plan.profile_read(reset=True)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    accepted = sum(1 for h in hist if h["gamma"] > 0)
    # metric: accepted CG iterations only (a line-search failure, gamma = 0, still costs its sweeps)
    value = frames * accepted / (ms / 1e3)

    # ---- roofline.  Per pass, from the CUDA events of the profiled run:
    #   algorithmic bytes = 8(a)'s per-frame figure x frames, flops = the implemented schedule's
    #   5 L log2 L count; the binding roof of a pass is max(bytes / BW, flops / P_FP32).
    bw, sm_mhz_max, src = peaks()
    fp = fp32_peak(local)
    p32 = fp["ffma_tflops"]
    A = 8.0 * cfg.npad ** 2
    prof_frames = (solver.sweeps - sw0 - sweeps) * (K_total // world) * cfg.nz if K_total else 0
    passes = {}
    for k, v in prof.items():
        if not v["launches"]:
            continue
        sec = v["ms"] / 1e3
        e = {"ms_per_step": v["ms"] / args.steps, "launches": v["launches"],
             "model_GBps": v["bytes"] / sec / 1e9, "TFLOPs": v["flops"] / sec / 1e12,
             "fp32_frac": v["flops"] / sec / 1e12 / p32}
        if k in ALG_BYTES_A and prof_frames:
            ab = ALG_BYTES_A[k] * A * prof_frames
            e.update({"alg_bytes_per_frame": ALG_BYTES_A[k] * A, "alg_GBps": ab / sec / 1e9,
                      "hbm_frac": ab / sec / 1e9 / bw,
                      "binding_frac": max(ab / (bw * 1e9), v["flops"] / (p32 * 1e12)) / sec,
                      "us_per_frame": 1e6 * sec / prof_frames, "flops_per_frame": v["flops"] / prof_frames})
        passes[k] = e
    chain = [k for k in ALG_BYTES_A if k in passes]
    top = max(chain or passes, key=lambda k: prof[k]["ms"])
    P = prof[top]
    nl = max(P["launches"], 1)
    launch_s = P["ms"] / 1e3 / nl
    fl_launch = P["flops"] / nl
    frames_per_launch = prof_frames / nl if (top in ALG_BYTES_A and prof_frames) else None
    by_launch = ALG_BYTES_A.get(top, 0) * A * frames_per_launch if frames_per_launch else P["bytes"] / nl
    t_hbm, t_alu = by_launch / (bw * 1e9), fl_launch / (p32 * 1e12)
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        try:
            tj = json.load(open(tfile))
            if tj.get("_workload") == cfg.name and top in tj:  # ncu dram bytes per launch of the same launch shape
                traffic = tj[top]
        except Exception:
            traffic = None
    if t_hbm >= t_alu:
        roof = {"bound": "hbm", "achieved": by_launch / launch_s / 1e9, "peak": bw, "unit": "GB/s"}
    else:
        roof = {"bound": "alu", "achieved": fl_launch / launch_s / 1e12, "peak": p32, "unit": "TFLOP/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof.update({"traffic": traffic, "kernel": top,
                 "peak_source": f"hbm: {src} MEASURED_PEAKS.json {bw:.0f} GB/s; fp32: {fp['source']} "
                                f"{p32:.1f} TFLOP/s at {fp['sm_mhz']:.0f} MHz",
                 "alg_bytes_per_launch": by_launch, "flops_per_launch": fl_launch,
                 "frames_per_launch": frames_per_launch, "launch_us": 1e6 * launch_s,
                 "hbm_frac": by_launch / launch_s / 1e9 / bw, "fp32_frac": fl_launch / launch_s / 1e12 / p32,
                 "traffic_over_alg": (traffic / by_launch) if traffic else None,
                 "share_of_step": P["ms"] / ms_prof})
    # step level: T_roof = frames x max(B_min / BW, F_alg / P_FP32) against the measured step
    f_alg = sum(passes[k].get("flops_per_frame", 0) for k in chain)
    t_frame = (ms / 1e3) / (frames * max(accepted, 1)) if frames else None  # ms spans all timed steps
    step = None
    if frames and f_alg:
        t_roof = max(B_MIN_A * A / (bw * 1e9), f_alg / (p32 * 1e12))
        step = {"B_min_bytes_per_frame": B_MIN_A * A, "F_alg_flops_per_frame": f_alg,
                "T_roof_us_per_frame": 1e6 * t_roof, "T_meas_us_per_frame": 1e6 * t_frame,
                "binding_frac": t_roof / t_frame,
                "binding": "fp32" if f_alg / (p32 * 1e12) > B_MIN_A * A / (bw * 1e9) else "hbm",
                "hbm_frac_B_min": B_MIN_A * A * value / 1e9 / bw,
                "hbm_frac_B_min_8TBps": B_MIN_A * A * value / 1e9 / 8000.0}
    prof_overhead = ms_prof / ms - 1.0
    # ---- e2e: same metric through the public API with the step's input (sqrt d) copied
    #      from pinned host memory every step and the step's result (F) read back
    e2e = None
    if not args.no_e2e:
        host_d = torch.empty(sqrt_d.shape, dtype=torch.float32, pin_memory=True)
        host_d.copy_(sqrt_d)
        ns = max(1, min(args.steps, 3))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sw1 = solver.sweeps
        e0.record()
        stage = hasattr(plan, "stage_sqrt_d")
        for _ in range(ns):
            if stage:  # holo_stage_sqrt_d(ref): streamed per angle / frame batch inside the step's first sweep
                (plan.stage_sqrt_dref if cfg.name == "cfg4" else plan.stage_sqrt_d)(host_d, sqrt_d)
            else:
                sqrt_d.copy_(host_d, non_blocking=True)
            solver.iterate()  # ends with the D2H read of F and the dots
        e1.record()
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e_sweeps = solver.sweeps - sw1
        e2e = {"value": frames * ns / (float(te.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(sqrt_d.numel() * 4), "d2h_bytes_per_step": int(40 * e_sweeps / ns),
               "steps": ns, "h2d": "holo_stage_sqrt_d(ref): per angle (reference-frame) batch on a copy stream, overlapped with the "
                                   "sweep" if stage else "one copy before the step"}
        del host_d

    # ---- the multiresolution schedule: 3 levels (4x4, 2x2, 1x1 binning)
    #      of the same workload on a smaller angle set, timed with CUDA events per level (a separate
    #      run after the headline measurement, its own memory: the main solver is released first)
    multires = None
    if args.multires_angles > 0 and cfg.name != "cfg4":
        del solver, plan, sqrt_d
        torch.cuda.empty_cache()
        multires = run_multires(args, cfg, hb, dev, local, k0)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_ref(cfg) if cfg.name == "cfg4" else cpu_baseline(cfg)

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "c64 (fp32 complex; fp64 reductions)", "data": "synthetic",
            "config": conf,
            "iterations": args.steps, "accepted_iterations": accepted,
            "sweeps_per_step": sweeps / args.steps, "sweeps_per_s": sweeps / (ms / 1e3),
            "F_last": hist[-1]["F"], "gamma_last": hist[-1]["gamma"],
            "roofline_step": step, "fp32_peak": fp,
            "profiled_steps_overhead": prof_overhead,
            "roofline": roof, "passes": passes, "gpu_launches": int(launches),
            "clocks": clocks, "e2e": e2e, "cpu_baseline": cpu, "multires": multires,
        }
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
