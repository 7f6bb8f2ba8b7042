"""Probe: do two independent half-size node groups on two streams beat one full-size launch
sequence?  One C4_G1 context (8 nodes, 90 angles) against two 4-node / 45-angle contexts run
concurrently on two streams (same per-node work: 1024^2, ~11 angles, CG5, K-means 64)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from dataclasses import replace
import torch
from paper_2410_06106_b200 import configs as C, tomoq

def make(cfg):
    inp = C.make_inputs(cfg, with_truth=False)
    ctx = tomoq.Context(cfg.N, cfg.n_angles, cfg.n_det, cfg.nodes, inp.edges, split=cfg.split, rule=cfg.rule)
    ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1)
    ctx.set_quantizer(cfg.quant, k=cfg.k, lloyd=cfg.lloyd)
    ctx.set_sinogram(0, inp.sino[0])
    return ctx

full = C.C4(1)
half = replace(full, nodes=4, n_angles=45, graph="ring")
c8 = make(full)
h1, h2 = make(half), make(half)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
it = 48
for c, s in ((c8, s1), (h1, s1), (h2, s2)):
    c.run(8, s)
torch.cuda.synchronize()

def timed(fn, s):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s); fn(); b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it

for rep in range(3):
    t8 = timed(lambda: c8.run_async(it, s1), s1)
    th = timed(lambda: h1.run_async(it, s1), s1)
    def both():
        ev = torch.cuda.Event(); ev.record(s1); s2.wait_event(ev)
        h1.run_async(it, s1); h2.run_async(it, s2)
        ev2 = torch.cuda.Event(); ev2.record(s2); s1.wait_event(ev2)
    tb = timed(both, s1)
    def c8_steps():
        for _ in range(it):
            c8.run_async(1, s1)
    def lock():  # one iteration of each half per step, joined after every step (as a dual would)
        for _ in range(it):
            ev = torch.cuda.Event(); ev.record(s1); s2.wait_event(ev)
            h1.run_async(1, s1); h2.run_async(1, s2)
            ev2 = torch.cuda.Event(); ev2.record(s2); s1.wait_event(ev2)
    t8s = timed(c8_steps, s1)
    tl = timed(lock, s1)
    print(f"8-node ctx {t8:.4f} ms/iter | one 4-node ctx {th:.4f} | two 4-node ctxs concurrently {tb:.4f} "
          f"(x{t8 / tb:.3f} vs 8-node) | per-iteration launches: 8-node {t8s:.4f}, two halves joined every "
          f"iteration {tl:.4f} (x{t8s / tl:.3f})", flush=True)
for c in (c8, h1, h2):
    c.wait(); c.close()
