import sys, time, torch
sys.path.insert(0, '/root/repo')
import synth, numpy as np
import paper_2407_20304_b200 as hb
from paper_2407_20304_b200.solver import JointCG
cfg = synth.CONFIGS['cfg3']; K = 16
dev = torch.device('cuda', 0)
def T(): torch.cuda.synchronize(); return time.perf_counter()
for rep in range(2):
    t0 = T()
    plan = hb.Plan(cfg.n, cfg.npad, cfg.z1, K, cfg.wavelength, cfg.Z, cfg.det_pixel, device=0, angle_batch=8)
    t1 = T()
    plan.set_shifts(synth.shifts(cfg)[:K]); t2 = T()
    q_t = synth.probe(cfg, device=dev, dtype=torch.complex64)
    psi_t = synth.psi_stack(cfg, K=K, device=dev, dtype=torch.complex64)
    w = torch.empty(K, cfg.nz, cfg.n, cfg.n, dtype=torch.complex64, device=dev)
    t3 = T(); plan.fwd(psi_t, q_t, w); t4 = T()
    d = w.abs().float().contiguous(); del w
    cg = JointCG(plan, d, torch.ones_like(psi_t), 0.9 * q_t, rho_q=1.0 / K)
    t5 = T(); cg.start(); t6 = T()
    for _ in range(3): cg.iterate()
    t7 = T()
    print(f"rep {rep}: plan {1e3*(t1-t0):.0f} ms, shifts {1e3*(t2-t1):.0f}, fwd {1e3*(t4-t3):.0f}, start {1e3*(t6-t5):.0f}, 3 it {1e3*(t7-t6):.0f} ms sweeps {cg.sweeps}", flush=True)
    del cg, plan, d, psi_t
    torch.cuda.empty_cache()
