import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2410_06106_b200 import configs as C, tomoq
cfg = C.C4(1)
inp = C.make_inputs(cfg, with_truth=False)
ctx = tomoq.Context(cfg.N, cfg.n_angles, cfg.n_det, cfg.nodes, inp.edges, split=cfg.split, rule=cfg.rule)
ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1)
ctx.set_quantizer(cfg.quant, k=cfg.k, lloyd=cfg.lloyd)
sino = torch.from_numpy(inp.sino[0]).pin_memory()
img = [torch.empty(cfg.N * cfg.N, dtype=torch.float32).pin_memory() for _ in range(2)]
ctx.set_sinogram(0, sino)
st, cs = torch.cuda.Stream(), torch.cuda.Stream()
ctx.run(5, st); torch.cuda.synchronize()
for mode in ("overlap", "sync-before-set"):
    ts = []
    for rep in range(8):
        t0 = time.perf_counter(); ctx.set_sinogram(0, sino); t1 = time.perf_counter()
        ctx.run(1, st); t2 = time.perf_counter()
        ctx.image_async(img[rep & 1], cs, 0, 0)
        if mode != "overlap": cs.synchronize()
        t3 = time.perf_counter()
        ts.append((t1 - t0, t2 - t1, t3 - t2))
    cs.synchronize()
    import statistics
    print(mode, [round(1e3 * statistics.median(x), 3) for x in zip(*ts)])
# H2D alone timing
t0 = time.perf_counter()
for _ in range(10): ctx.set_sinogram(0, sino)
print("set_sinogram alone", (time.perf_counter() - t0) * 100, "ms")
