"""Where the end-to-end loop loses time vs device-only replay (run on a GPU box)."""
import sys, time, statistics
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
K = 40
def loop(name, do_set, do_img, asyn=True):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    t00 = time.perf_counter()
    e0.record(st)
    for k in range(K):
        t0 = time.perf_counter()
        if do_set: ctx.set_sinogram(0, sino)
        t1 = time.perf_counter()
        if asyn: ctx.run_async(1, st)
        else: ctx.run(1, st)
        t2 = time.perf_counter()
        if do_img: ctx.image_async(img[k & 1], cs, 0, 0)
        t3 = time.perf_counter()
        ts.append((t1 - t0, t2 - t1, t3 - t2))
    ctx.wait(); cs.synchronize()
    e1.record(st); torch.cuda.synchronize()
    wall = (time.perf_counter() - t00) * 1e3 / K
    print(f"{name:28s} wall/step {wall:.3f} ms  dev/step {e0.elapsed_time(e1)/K:.3f}  host med (set, run, img) ms",
          [round(1e3 * statistics.median(x), 3) for x in zip(*ts)], flush=True)
def loop2(name, fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for k in range(K):
        ctx.run_async(1, st)
        fn(k)
    ctx.wait(); cs.synchronize()
    e1.record(st); torch.cuda.synchronize()
    print(f"{name:28s} dev/step {e0.elapsed_time(e1)/K:.3f}", flush=True)
small = torch.zeros(1024, device="cuda")
big = torch.zeros(cfg.N * cfg.N, device="cuda")
def f_small(k):
    with torch.cuda.stream(st): small.add_(1.0)
def f_big(k):
    with torch.cuda.stream(st): big.add_(1.0)
def f_d2h(k):
    ev = torch.cuda.Event(); ev.record(st); cs.wait_event(ev)
    with torch.cuda.stream(cs): img[k & 1].copy_(big, non_blocking=True)
def f_h2d(k):
    with torch.cuda.stream(cs): big.copy_(img[k & 1], non_blocking=True)
loop2("async + small kernel", f_small)
loop2("async + 4MB kernel", f_big)
loop2("async + d2h 4MB (copy st)", f_d2h)
loop2("async + h2d 4MB (copy st)", f_h2d)
loop("run_async only", False, False)
loop("run (sync) only", False, False, asyn=False)
loop("async + set", True, False)
loop("async + img", False, True)
loop("async + set + img", True, True)
loop("sync + set + img", True, True, asyn=False)
