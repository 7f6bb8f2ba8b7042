"""Every kernel family through the C-ABI at small sizes, writing the results to an .npz file:
config 1 (graph rule, CG5; paper and consensus rules; Siddon projector; fp64 GD), config 2's
structure at 128^2 (K-means 16: bit-planes, DSMEM cluster Lloyd), config 3's structure at 64^2
(DCT, JPEG entropy coding), two slices of config 5's structure (alternating codecs), world 2
over the loopback transport, the stateless entry points.

tests/test_gpu_guard.py runs it twice -- plainly and with TQ_GUARD=1 (guard bands around
every device allocation, checked after every run; allocations poisoned with 0xff) -- and
requires bitwise equal results and intact guards: the stand-in for compute-sanitizer's
memcheck / initcheck, which is closed on the GPU pool.

python tools/guard_run.py OUT.npz"""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_06106_b200 import configs as C  # noqa: E402
from paper_2410_06106_b200 import tomoq  # noqa: E402
from tests.cases import gpu_context  # noqa: E402

OUT = {}


def run(name, cfg, iters=3, precision=0):
    inp = C.make_inputs(cfg, with_truth=False)
    ctx = gpu_context(cfg, inp, precision=precision, keep_labels=cfg.quant != C.Q_NONE)
    ctx.run(iters)
    for s in range(len(inp.sino)):
        OUT[f"{name}_s{s}"] = np.stack([ctx.image(s, m) for m in range(cfg.nodes)])
        OUT[f"{name}_state{s}"] = ctx.export_state(s, 0)
    ctx.close()
    tomoq.debug_guard_check()
    print(name, "ok", flush=True)


def loopback(name, cfg, world=2, iters=3):
    inp = C.make_inputs(cfg, with_truth=False)
    lid = tomoq.loopback_id()
    imgs = {}

    def worker(r):
        ctx = tomoq.Context(cfg.N, cfg.n_angles, cfg.n_det, cfg.nodes, inp.edges, split=cfg.split, rule=cfg.rule,
                            rank=r, world=world, nccl_id=lid)
        ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1)
        ctx.set_quantizer(cfg.quant, k=cfg.k, lloyd=cfg.lloyd, quality=cfg.quality)
        ctx.set_sinogram(0, inp.sino[0])
        ctx.run(iters)
        for m in range(r, cfg.nodes, world):
            imgs[m] = ctx.image(0, m)
        ctx.close()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    OUT[name] = np.stack([imgs[m] for m in range(cfg.nodes)])
    tomoq.debug_guard_check()
    print(name, "ok", flush=True)


def main(path):
    run("c1", C.C1())
    for rule, nm in ((C.RULE_PAPER, "paper"), (C.RULE_CONSENSUS, "consensus")):
        cfg = C.C1()
        cfg.rule = rule
        run(nm, cfg)
    run("c2", C.scaled(C.C2(), 128, 96))
    cfg = C.scaled(C.C3(), 64, 96)
    run("c3", cfg)
    cfg.jpeg_restart = 4
    run("c3_jpeg", cfg)
    run("c5", C.scaled(C.C5(slices=2), 64, 96))
    cfg = C.C1()
    cfg.projector = 1
    run("siddon", cfg)
    cfg = C.C1()
    cfg.inner, cfg.e1 = C.INNER_GD, 3
    run("gd_fp64", cfg, precision=1)
    loopback("loop_c2", C.scaled(C.C2(), 128, 96))
    # node groups (concurrent chains; the small images need TQ_GROUPS to enable them)
    for nm, cfg, g in (("c2_groups", C.scaled(C.C2(), 128, 96), "4"), ("c3_groups", C.scaled(C.C3(), 64, 96), "8"),
                       ("c5_groups", C.scaled(C.C5(slices=2), 64, 96), "4")):
        os.environ["TQ_GROUPS"] = g
        run(nm, cfg)
    os.environ.pop("TQ_GROUPS", None)
    x = torch.rand(64, 64, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3))
    s = tomoq.project(x, 90, 91)
    OUT["stateless_fp"] = s.cpu().numpy()
    OUT["stateless_bp"] = tomoq.backproject(s, 64, 90).cpu().numpy()
    cen, planes, lab = tomoq.kmeans_encode(x.view(-1), 8, 5)
    OUT["stateless_km"] = lab.cpu().numpy()
    coef, mm = tomoq.dct_encode(x, 50)
    OUT["stateless_dct"] = coef.cpu().numpy()
    torch.cuda.synchronize()
    tomoq.debug_guard_check()
    np.savez(path, **OUT)
    print("all ok", flush=True)


if __name__ == "__main__":
    main(sys.argv[1])
