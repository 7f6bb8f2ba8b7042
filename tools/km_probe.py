"""Time the K-means encode component (tq_launch_component 3) of the C4_G1 context for
several Lloyd iteration counts (GPU box): python tools/km_probe.py"""
import torch

from paper_2410_06106_b200 import configs as C
from tests.cases import gpu_context

cfg = C.C4(1)
inp = C.make_inputs(cfg, with_truth=False)
for lloyd in (0, 1, 10, 20):
    cfg.lloyd = lloyd
    ctx = gpu_context(cfg, inp)
    ctx.run(2)
    s = torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.launch_component(3, 3, s.cuda_stream)
    s.synchronize()
    e0.record(s)
    ctx.launch_component(3, 20, s.cuda_stream)
    e1.record(s)
    s.synchronize()
    print(f"lloyd={lloyd:3d}: kmeans encode {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
    ctx.close()
