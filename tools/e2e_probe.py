"""Time each public-API call of the bench's end-to-end loop (diagnostic, GPU box)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_06106_b200 import configs as C, tomoq  # noqa: E402

cfg = C.C4(1)
inp = C.make_inputs(cfg, with_truth=False)
ctx = tomoq.Context(cfg.N, cfg.n_angles, cfg.n_det, cfg.nodes, inp.edges, split=cfg.split, rule=cfg.rule)
ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1)
ctx.set_quantizer(cfg.quant, k=cfg.k, lloyd=cfg.lloyd)
sino = torch.from_numpy(inp.sino[0]).pin_memory()
img = [torch.empty(cfg.N * cfg.N, dtype=torch.float32).pin_memory() for _ in range(2)]
ctx.set_sinogram(0, sino)
st, cs = torch.cuda.Stream(), torch.cuda.Stream()
ctx.run(5, st)
torch.cuda.synchronize()
for rep in range(6):
    t0 = time.perf_counter(); ctx.set_sinogram(0, sino); t1 = time.perf_counter()
    ctx.run(1, st); t2 = time.perf_counter()
    ctx.image_async(img[rep & 1], cs, 0, 0); t3 = time.perf_counter()
    print(f"set_sinogram {1e3*(t1-t0):.3f} ms  run(1) {1e3*(t2-t1):.3f} ms  image_async {1e3*(t3-t2):.3f} ms "
          f"device {ctx.stats()['ms_last_run']:.3f} ms")
cs.synchronize()
t0 = time.perf_counter(); ctx.run(20, st); torch.cuda.synchronize(); print("run(20)", (time.perf_counter()-t0)*1e3/20, "ms/iter")
