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
    return {"value": 1.0 / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"1 frame (k={k}, j={j}) of {cfg.name}: F + grad_psi + grad_q term on the "
                      f"{cfg.npad}^2 torus, numpy/BLAS fp64 oracle (oracle/np_oracle.py); {dt:.2f} s"}


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
        plan = hb.Plan(cfg.n, cfg.npad, cfg.z1, K, cfg.wavelength, cfg.Z, cfg.det_pixel, device=local)
        plan.set_shifts(synth.shifts(cfg)[k0:k0 + K] if k0 + K <= cfg.n_angles else
                        np.resize(synth.shifts(cfg), (k0 + K, cfg.nz, 2))[k0:k0 + K])
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
                "npad": cfg.npad, "rho_q": rho_q, "parallelism": f"angle-sharded dp{world}",
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
    value = frames * args.steps / (ms / 1e3)

    # ---- roofline of the dominant kernel (CUDA events on the plan's stream, same region)
    bw, sm_mhz_max, src = peaks()
    fp32_peak = N_SM * FP32_LANES_PER_SM * 2 * sm_mhz_max * 1e6 / 1e12  # TFLOP/s
    top = max(prof, key=lambda k: prof[k]["ms"])
    P = prof[top]
    sec = P["ms"] / 1e3
    gbs = P["bytes"] / sec / 1e9
    tfs = P["flops"] / sec / 1e12
    t_hbm, t_alu = P["bytes"] / (bw * 1e9), P["flops"] / (fp32_peak * 1e12)
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get(top)
        except Exception:
            traffic = None
    if t_hbm >= t_alu:
        roof = {"bound": "hbm", "achieved": gbs, "peak": bw, "unit": "GB/s", "frac": gbs / bw, "traffic": traffic}
    else:
        roof = {"bound": "alu", "achieved": tfs, "peak": fp32_peak, "unit": "TFLOP/s", "frac": tfs / fp32_peak,
                "traffic": traffic}
    roof.update({"kernel": top, "peak_source": f"{src} (hbm {bw:.0f} GB/s; fp32 = 148 SM x 128 x 2 x "
                 f"{sm_mhz_max:.0f} MHz)", "share_of_step": P["ms"] / ms_prof,
                 "bytes_per_launch": P["bytes"] / max(P["launches"], 1),
                 "flops_per_launch": P["flops"] / max(P["launches"], 1),
                 "launch_us": 1e3 * P["ms"] / max(P["launches"], 1)})
    tot_bytes = sum(v["bytes"] for v in prof.values())
    prof_overhead = ms_prof / ms - 1.0
    passes = {k: {"ms_per_step": v["ms"] / args.steps, "launches": v["launches"],
                  "GBps": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] > 0 else 0,
                  "TFLOPs": (v["flops"] / (v["ms"] / 1e3) / 1e12) if v["ms"] > 0 else 0}
              for k, v in prof.items() if v["launches"]}

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
        for _ in range(ns):
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
               "steps": ns}
        del host_d

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_ref(cfg) if cfg.name == "cfg4" else cpu_baseline(cfg)

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "c64 (fp32 complex; fp64 reductions)", "data": "synthetic",
            "config": conf,
            "sweeps_per_step": sweeps / args.steps,
            "F_last": hist[-1]["F"], "gamma_last": hist[-1]["gamma"],
            "hbm_frac_step": (tot_bytes / (ms_prof / 1e3) / 1e9) / bw,
            "profiled_steps_overhead": prof_overhead,
            "roofline": roof, "passes": passes, "gpu_launches": int(launches),
            "clocks": clocks, "e2e": e2e, "cpu_baseline": cpu,
        }
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
