"""Upper bound for per-node dependencies across iterations: eight 1-node contexts (C4 per-node work:
1024^2, 11-12 angles, CG5, K-means 64) on eight streams, free-running vs joined after every
iteration, against the 8-node C4_G1 context (node groups on)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from dataclasses import replace
import torch
from paper_2410_06106_b200 import configs as C, tomoq

def make(cfg, edges=None):
    inp = C.make_inputs(cfg, with_truth=False)
    ctx = tomoq.Context(cfg.N, cfg.n_angles, cfg.n_det, cfg.nodes, inp.edges if edges is None else edges,
                        split=cfg.split, rule=cfg.rule)
    ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1)
    ctx.set_quantizer(cfg.quant, k=cfg.k, lloyd=cfg.lloyd)
    ctx.set_sinogram(0, inp.sino[0])
    return ctx

full = C.C4(1)
one = replace(full, nodes=1, n_angles=11, graph="ring")
c8 = make(full)
cs = [make(one, edges=[]) for _ in range(8)]
ss = [torch.cuda.Stream() for _ in range(8)]
it = 48
c8.run(8, ss[0])
for c, s in zip(cs, ss):
    c.run(8, s)
torch.cuda.synchronize()

def timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(ss[0]); fn(); b.record(ss[0])
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it

def fork():
    ev = torch.cuda.Event(); ev.record(ss[0])
    for s in ss[1:]:
        s.wait_event(ev)

def join():
    for s in ss[1:]:
        ev = torch.cuda.Event(); ev.record(s); ss[0].wait_event(ev)

def free():
    fork()
    for c, s in zip(cs, ss):
        c.run_async(it, s)
    join()

def lock():
    for _ in range(it):
        fork()
        for c, s in zip(cs, ss):
            c.run_async(1, s)
        join()

for rep in range(3):
    t8 = timed(lambda: c8.run_async(it, ss[0]))
    tf = timed(free)
    tl = timed(lock)
    print(f"8-node ctx {t8:.4f} ms/iter | eight 1-node ctxs free-running {tf:.4f} | joined every iteration {tl:.4f}",
          flush=True)
for c in [c8] + cs:
    c.wait(); c.close()
