import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2410_06106_b200 import configs as C
from tests.cases import oracle_case
cfg = C.C4(1)
inp = C.make_inputs(cfg, with_truth=False)
print("cpus", os.cpu_count(), flush=True)
for th in (8, 1):
    o = oracle_case(cfg, inp, threads=th)
    o.run(1)
    t0 = time.perf_counter(); o.run(2); dt = time.perf_counter() - t0
    print("threads", th, "s per iteration", round(dt / 2, 3), flush=True)
