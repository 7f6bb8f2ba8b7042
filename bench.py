"""Benchmark of the hot path: decentralized quantized ADMM iterations (Alg. 4
with K-means quantized exchange) on BASELINE.json config 4 (weak scaling: 8 ADMM
nodes per GPU, 1024^2 image, 90 angles per GPU, random 4-regular graph, CG5, K=64).

One "step" = one ADMM iteration of every node: E1+1 forward/back projector pairs
(CG), the K-means encode of every node's iterate, the exchange (NCCL send/recv of
payloads along cross-GPU edges), decode and the dual/rhs update.

python bench.py [--gpus N --steps K --warmup W] [--impl reference]
Prints ONE JSON line (rank 0).  See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ADMM iterations/s and projector Gvoxel-updates/s vs HBM roofline, 1/2/4/8 GPU"
UNIT = "GVU/s"
LSU_VU_PER_CLK_SM = 16  # 2 fp32 taps per VU through a 128 B/clk/SM L1/smem path


def env_int(k, d):
    return int(os.environ.get(k, d))


def peaks():
    p = {"hbm_gbs": None, "sm_max_mhz": None, "src": "fallback"}
    try:
        m = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        p.update(hbm_gbs=m["hbm_gbs"], sm_max_mhz=m["sm_max_mhz"], src="measured")
    except Exception:
        p.update(hbm_gbs=6650.0, sm_max_mhz=1965.0)
    return p


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.proc, self.out = device, None, ""

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def vu_per_iter(cfg):
    """voxel-updates per ADMM iteration over all nodes, counted algorithmically (the same
    count for both arms and every round): the standard CG formulation's (E1+1) A/A^T pairs
    (residual + E1 steps), each N^2 x (angles of the node) VU; summed over nodes = N^2 x
    n_angles.  The CUDA path executes one backprojection fewer per
    solve (the last step's r update is never used): see projector_applications."""
    apps = (cfg.e1 + 1) if cfg.inner == 1 else cfg.e1
    return 2 * apps * cfg.N * cfg.N * cfg.n_angles * cfg.slices


AX_MAXAGE = 16  # the engine's refresh period of the kept A x (TQ_AX_MAXAGE)


def projector_applications(cfg):
    """(algorithmic, executed) projector applications (A or A^T) per ADMM iteration.  CG on the
    graph rule executes E1 forward projections (the residual's A x is kept, one refresh per
    AX_MAXAGE iterations) and E1 backprojections (residual + E1 - 1 steps)."""
    if cfg.inner == 1:
        return 2 * (cfg.e1 + 1), 2 * cfg.e1 + 1.0 / AX_MAXAGE
    return 2 * cfg.e1, 2 * cfg.e1


def sm_count():
    import torch
    return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count


def host_info():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"host_cores": os.cpu_count(), "host_model": model}


def c5_iteration(tomoq, torch, stream, slices=4, iters=3):
    """Config 5 whole ADMM iterations at G = 1 on `slices` of its 32 slices (2048^2, 1500
    angles, 8 nodes per slice on a complete graph, CG5, even slices K-means 32 / odd slices DCT
    q75): ms per iteration and G VU/s, CUDA events over `iters` iterations after one warm-up."""
    from paper_2410_06106_b200 import configs as C
    cfg = C.C5(slices=slices)
    inp = C.make_inputs(cfg, with_truth=False)
    ctx = tomoq.Context(cfg.N, cfg.n_angles, cfg.n_det, cfg.nodes, inp.edges, split=cfg.split, rule=cfg.rule,
                        n_slices=slices)
    ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1)
    ctx.set_quantizer(cfg.quant, k=cfg.k, lloyd=cfg.lloyd, quality=cfg.quality)
    for s_, d in enumerate(inp.sino):
        ctx.set_sinogram(s_, d)
    ctx.run(1, stream)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    ctx.run(iters, stream)
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / iters
    ctx.close()
    vu = vu_per_iter(cfg)
    return {"workload": f"C5 at G = 1: {slices} of its 32 slices (2048^2, 1500 angles, 8 nodes per slice, "
                        f"K-means 32 / DCT q75 by slice), {iters} timed iterations",
            "ms_per_iter": ms, "gvu_s": vu / (ms / 1e3) / 1e9,
            "ms_per_iter_32_slices_extrapolated": ms * 32 / slices}


def projector_c5_geometry(tomoq, torch, stream, reps=5):
    """Forward projector and CG backprojector on one C5 slice's geometry: 2048^2 image,
    1500 angles, 8 nodes of 187-188 angles on one GPU (random sinogram: timing only)."""
    from paper_2410_06106_b200 import configs as C
    from paper_2410_06106_b200 import synth
    cfg = C.C5(slices=1)
    ctx = tomoq.Context(cfg.N, cfg.n_angles, cfg.n_det, cfg.nodes, synth.complete(cfg.nodes), split=cfg.split,
                        rule=cfg.rule)
    ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1)
    ctx.set_quantizer(tomoq.Q_NONE)
    sino = torch.rand(cfg.n_angles, cfg.n_det, device="cuda")
    ctx.set_sinogram(0, sino)
    out = {"workload": "C5 slice geometry: N=2048, 1500 angles, 2897 bins, 8 nodes x 187-188 angles"}
    peak = LSU_VU_PER_CLK_SM * sm_count() * peaks()["sm_max_mhz"] * 1e6 / 1e9
    for comp, name in ((0, "fp"), (1, "bp_cgr")):
        ctx.launch_component(comp, 2, stream)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        units = ctx.launch_component(comp, reps, stream)
        b.record(stream)
        torch.cuda.synchronize()
        t = a.elapsed_time(b) / reps
        out[name] = {"ms": t, "gvu_s": units / (t / 1e3) / 1e9, "frac": units / (t / 1e3) / 1e9 / peak}
    ctx.close()
    return out


def projector_siddon_c4(tomoq, torch, stream, reps=10):
    """NEXT-3 measurement: the Siddon projector (exact intersection lengths, R-26) on the
    bench workload's geometry (C4_G1: 1024^2, 90 angles, 8 nodes), forward and CG
    backprojector timed like the roofline components, next to Joseph."""
    from paper_2410_06106_b200 import configs as C
    cfg = C.C4(1)
    inp = C.make_inputs(cfg, with_truth=False)
    out = {"workload": "C4_G1 geometry with the Siddon projector"}
    peak = LSU_VU_PER_CLK_SM * sm_count() * peaks()["sm_max_mhz"] * 1e6 / 1e9
    for proj, name in ((tomoq.PROJ_SIDDON, "siddon"), (tomoq.PROJ_JOSEPH, "joseph")):
        ctx = tomoq.Context(cfg.N, cfg.n_angles, cfg.n_det, cfg.nodes, inp.edges, split=cfg.split, rule=cfg.rule,
                            projector=proj)
        ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1)
        ctx.set_quantizer(tomoq.Q_NONE)
        ctx.set_sinogram(0, torch.tensor(inp.sino[0], device="cuda"))
        ctx.run(1)
        res = {}
        for comp, cname in ((0, "fp"), (1, "bp_cgr")):
            ctx.launch_component(comp, 2, stream)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            units = ctx.launch_component(comp, reps, stream)
            b.record(stream)
            torch.cuda.synchronize()
            t = a.elapsed_time(b) / reps
            res[cname] = {"us": t * 1e3, "gvu_s": units / (t / 1e3) / 1e9, "frac": units / (t / 1e3) / 1e9 / peak}
        ctx.run(5)
        res["admm_iter_ms"] = ctx.stats()["ms_last_run"] / 5
        out[name] = res
        ctx.close()
    return out


def dct_entropy_c3(tomoq, torch, stream, reps=10, restart=4):
    """NEXT-2 measurement on config 3 as stated (16 nodes x 512^2, 4x4 torus, DCT q50):
    the DCT-J encode stage (tq_launch_component 4: min/max, integer DCT, quantisation and,
    with JPEG entropy coding, Huffman coding of every local payload) timed with events,
    and the payload bytes per ADMM iteration with and without entropy coding (after 3
    iterations from zero, synthetic phantom data)."""
    from paper_2410_06106_b200 import configs as C
    cfg = C.C3()
    inp = C.make_inputs(cfg, with_truth=False)
    out = {"workload": "C3: 16 nodes x 512^2, DCT q50, restart interval %d blocks" % restart}
    for R in (0, restart):
        ctx = tomoq.Context(cfg.N, cfg.n_angles, cfg.n_det, cfg.nodes, inp.edges, split=cfg.split, rule=cfg.rule)
        ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1)
        ctx.set_quantizer(cfg.quant, quality=cfg.quality, jpeg_restart=R)
        ctx.set_sinogram(0, torch.tensor(inp.sino[0], device="cuda"))
        ctx.run(3)
        ctx.launch_component(4, 2, stream)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        units = ctx.launch_component(4, reps, stream)
        b.record(stream)
        torch.cuda.synchronize()
        t = a.elapsed_time(b) / reps
        key = "entropy" if R else "plain"
        out[key] = {"encode_us": t * 1e3, "pixels_per_s": units / (t / 1e3),
                    "payload_bytes_per_iter": ctx.stats()["payload_bytes_logical"]}
        ctx.close()
    out["compression_vs_plain"] = out["plain"]["payload_bytes_per_iter"] / out["entropy"]["payload_bytes_per_iter"]
    return out


def cpu_baseline(cfg_g1, iters=2):
    """The fp64 oracle as it stands, on the host cores, on a bounded sample: `iters`
    ADMM iterations of the per-GPU share of the workload (config 4 at G = 1), OpenMP over
    the nodes (node-level threads measured faster than nesting the projector's row loops
    under them; the row loops parallelise when a run has one node thread)."""
    from paper_2410_06106_b200 import configs as C
    from tests.cases import oracle_case
    inp = C.make_inputs(cfg_g1, with_truth=False)
    threads = min(cfg_g1.nodes, os.cpu_count() or 1)
    o = oracle_case(cfg_g1, inp, threads=threads)
    t0 = time.perf_counter()
    o.run(iters)
    dt = time.perf_counter() - t0
    return {"value": vu_per_iter(cfg_g1) * iters / dt / 1e9, "unit": UNIT, "cores": threads,
            "kind": "oracle", "sample": f"{iters} ADMM iterations of {cfg_g1.name} (8 nodes, 1024^2, "
                                        f"K-means 64), OpenMP over the {threads} nodes",
            "seconds": round(dt, 2), **host_info()}


def bench_config(cfg, world):
    """The `config` object of the JSON line (identical for both arms)."""
    return {"workload": cfg.name, "N": cfg.N, "nodes": cfg.nodes, "nodes_per_gpu": cfg.nodes // world,
            "n_angles": cfg.n_angles, "n_det": cfg.n_det, "graph": "random 4-regular",
            "inner": "CG5", "quantizer": "kmeans K=64 (10 Lloyd)", "rule": "graph",
            "parallelism": f"nodes interleaved over {world} GPU(s), NCCL send/recv of payloads; per GPU the "
                           f"nodes' inner solves + encodes as concurrent launch chains (node groups, DESIGN.md 6.1)",
            "l2": "no flush: per-GPU working set ~0.25 GB > 126 MB L2"}


def run_reference(args):
    """--impl reference: the oracle, rank 0 only."""
    rank, world = env_int("RANK", 0), env_int("WORLD_SIZE", 1)
    if rank != 0:
        return
    from paper_2410_06106_b200 import configs as C
    from tests.cases import oracle_case
    cfg = C.C4(1)  # bounded sample: the per-GPU share of C4_G<world> (8 nodes, 90 angles)
    inp = C.make_inputs(cfg, with_truth=False)
    threads = min(cfg.nodes, os.cpu_count() or 1)
    o = oracle_case(cfg, inp, threads=threads)
    o.run(args.warmup)
    t0 = time.perf_counter()
    o.run(args.steps)
    dt = time.perf_counter() - t0
    value = vu_per_iter(cfg) * args.steps / dt / 1e9
    sample = (f"each step = 1 ADMM iteration of {cfg.name} (the per-GPU share of C4_G{world}: 8 nodes, "
              f"1024^2, 90 angles, CG5, K-means 64) on the fp64 CPU oracle, OpenMP over the nodes")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / max(1, args.steps),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": bench_config(C.C4(world), world),
        "admm_iters_per_s": args.steps / dt,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample,
                         **host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c5-geometry", action="store_true")
    ap.add_argument("--precision", type=int, default=0)
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # `python bench.py --gpus N` without a launcher: one rank per GPU under torchrun
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if env_int("WORLD_SIZE", 1) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_int('WORLD_SIZE', 1)} "
                         f"(launch one rank per GPU, or drop the launcher and let bench.py spawn them)")
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    from paper_2410_06106_b200 import configs as C
    from paper_2410_06106_b200 import tomoq

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    assert args.warmup >= 3, "contract: W >= 3"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = C.C4(world)
    inp = C.make_inputs(cfg, with_truth=False)
    nid = None
    if world > 1:
        obj = [tomoq.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    ctx = tomoq.Context(cfg.N, cfg.n_angles, cfg.n_det, cfg.nodes, inp.edges, split=cfg.split,
                        rule=cfg.rule, rank=rank, world=world, nccl_id=nid, precision=args.precision,
                        device=local)
    ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1)
    ctx.set_quantizer(cfg.quant, k=cfg.k, lloyd=cfg.lloyd)
    sino_host = torch.from_numpy(inp.sino[0]).pin_memory()
    ctx.set_sinogram(0, sino_host)
    stream = torch.cuda.Stream(device=dev)  # a real stream (the legacy default stream has handle 0)
    torch.cuda.set_stream(stream)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up (also captures the CUDA graph of one iteration)
    ctx.run(args.warmup, stream)
    barrier()
    # ---- timed region: exactly K steps (ADMM iterations)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ctx.run(args.steps, stream)
    e1.record(stream)
    barrier()
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1))
    st = ctx.stats()
    vu_it = vu_per_iter(cfg)
    value = vu_it * args.steps / (ms / 1e3) / 1e9
    iters_per_s = args.steps / (ms / 1e3)

    # ---- end to end through the public API with host buffers: per step, H2D of the
    # slice sinogram from pinned memory (tq_set_sinogram), one iteration enqueued without
    # waiting (tq_run_async), D2H of a node's image (tq_get_image_async on a copy stream into
    # two pinned buffers), so the host work and the transfers of step k overlap the device
    # work of steps k - 1 and k + 1; tq_wait (divergence check) and every copy finish inside
    # the region
    img_host = [torch.empty(cfg.N * cfg.N, dtype=torch.float32).pin_memory() for _ in range(2)]
    copy_stream = torch.cuda.Stream()
    my_node = rank  # node `rank` lives on this rank (interleaved map)
    for k in range(max(args.warmup, 4)):  # untimed: the API path's lazily created buffers and events
        ctx.set_sinogram(0, sino_host)
        ctx.run_async(1, stream)
        ctx.image_async(img_host[k & 1], copy_stream, 0, my_node)
    ctx.wait()
    copy_stream.synchronize()
    barrier()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e2.record(stream)
    for k in range(args.steps):
        ctx.set_sinogram(0, sino_host)
        ctx.run_async(1, stream)
        ctx.image_async(img_host[k & 1], copy_stream, 0, my_node)
    ctx.wait()
    copy_stream.synchronize()
    e3.record(stream)
    barrier()
    e2e_ms = max_over_ranks(e2.elapsed_time(e3))
    e2e_wall = max_over_ranks((time.perf_counter() - t0) * 1e3)
    e2e_value = vu_it * args.steps / (max(e2e_ms, e2e_wall) / 1e3) / 1e9

    # ---- roofline of the dominant kernel (timed alone, CUDA events on this stream)
    pk = peaks()
    comp_ms, comp_units = {}, {}
    reps = 20
    for comp in (0, 1):
        ctx.launch_component(comp, 3, stream)
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        comp_units[comp] = ctx.launch_component(comp, reps, stream)
        b.record(stream)
        torch.cuda.synchronize()
        comp_ms[comp] = a.elapsed_time(b) / reps
    apps = {0: cfg.e1, 1: cfg.e1}  # forward projections (A x kept) / backprojections (E1 - 1 CG + 1 residual) per iteration
    share = {c: comp_ms[c] * apps[c] / (ms / args.steps) for c in comp_ms}
    dom = max(comp_ms, key=lambda c: comp_ms[c])
    names = {0: "forward projector A p (fp_persist_f32 tile pass + fp_reduce)",
             1: "backprojector A^T s + c p with the fused CG residual update r -= alpha q (bp_tile_kernel<float,CGR>)"}
    achieved = comp_units[dom] / (comp_ms[dom] / 1e3) / 1e9
    n_sm = sm_count()
    peak_vu = LSU_VU_PER_CLK_SM * n_sm * pk["sm_max_mhz"] * 1e6 / 1e9
    n_local = st["local_nodes"]
    compulsory = 4.0 * n_local * cfg.N ** 2 + 8.0 * (comp_units[dom] / cfg.N ** 2) * cfg.n_det
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = prof.get({0: "fp", 1: "bp"}[dom])
    except Exception:
        pass
    roofline = {
        "bound": "smem", "kernel": names[dom], "achieved": achieved, "peak": peak_vu, "unit": "GVU/s",
        "frac": achieved / peak_vu, "traffic": traffic,
        "peak_basis": f"shared-memory data path (l1tex shared wavefronts, measured 0.977/clk/SM in "
                      f"profiles/r1_smem_roofline.txt): 2 x 4-byte taps per VU at 128 B/clk/SM = {LSU_VU_PER_CLK_SM} "
                      f"VU/clk/SM x {n_sm} SMs x {pk['sm_max_mhz']} MHz (sm_max_mhz {pk['src']}); DESIGN.md section 6",
        "hbm_compulsory_gbs": compulsory / (comp_ms[dom] / 1e3) / 1e9, "hbm_peak_gbs": pk["hbm_gbs"],
        "share_of_step": share[dom],
        "components_ms": {"fp": comp_ms[0], "bp_cgr": comp_ms[1]},
    }

    # ---- the same projector kernels on config 5's node geometry (2048^2, 188 angles per node):
    # more angles per staged tile, so the per-tile staging is amortised (context, not the headline)
    c5_geom = None
    if rank == 0 and not args.no_c5_geometry:
        try:
            c5_geom = projector_c5_geometry(tomoq, torch, stream, reps=5)
        except Exception as exc:  # report, never fail the bench line
            c5_geom = {"error": str(exc)[:200]}
    # ---- config 5 whole iterations at G = 1 (a slice subset; context, not the headline)
    c5_iter = None
    if rank == 0 and world == 1 and not args.no_c5_geometry:
        try:
            c5_iter = c5_iteration(tomoq, torch, stream)
        except Exception as exc:
            c5_iter = {"error": str(exc)[:200]}
    # ---- NEXT-3: the Siddon projector on the bench geometry (context, not the headline)
    siddon_c4 = None
    if rank == 0 and not args.no_c5_geometry:
        try:
            siddon_c4 = projector_siddon_c4(tomoq, torch, stream)
        except Exception as exc:
            siddon_c4 = {"error": str(exc)[:200]}
    # ---- NEXT-2: JPEG entropy coding of the DCT payloads on config 3 (context, not the headline)
    jpeg_c3 = None
    if rank == 0 and not args.no_c5_geometry:
        try:
            jpeg_c3 = dct_entropy_c3(tomoq, torch, stream)
        except Exception as exc:
            jpeg_c3 = {"error": str(exc)[:200]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(C.C4(1))

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32" if args.precision == 0 else "f64",
            "data": "synthetic",
            "config": bench_config(cfg, world),
            "admm_iters_per_s": iters_per_s,
            "vu_per_step": vu_it,
            "projector_applications": dict(zip(("algorithmic", "executed"), projector_applications(cfg)),
                                           vu_basis="vu_per_step counts the algorithmic applications"),
            "roofline": roofline,
            "projector_c5_geometry": c5_geom,
            "c5_iteration": c5_iter,
            "dct_entropy_c3": jpeg_c3,
            "projector_siddon_c4": siddon_c4,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(sino_host.numel() * 4),
                    "d2h_bytes_per_step": int(cfg.N * cfg.N * 4), "ms_per_step": max(e2e_ms, e2e_wall) / args.steps},
            "gpu_launches": int(st["kernel_launches"]),
            "node_groups": int(st["node_groups"]),
            "clocks": clk,
            "payload_bytes_per_step": st["payload_bytes_logical"],
            "nccl_bytes_per_step_rank0": st["nccl_bytes_sent"],
        }
        print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
