"""NEXT-1: run the paper's experimental designs on workload W2 through the GPU path and
write profiles/r1_studies_<scale>.json plus a summary table (GPU box).

PYTHONPATH=. python tools/run_studies.py [--scale full|reduced] [--iters K]"""
import argparse
import json
import os
import time

from paper_2410_06106_b200 import studies

ap = argparse.ArgumentParser()
ap.add_argument("--scale", default="reduced", choices=["full", "reduced"])
ap.add_argument("--iters", type=int, default=None)
args = ap.parse_args()
t0 = time.perf_counter()
res = studies.studies(args.scale, args.iters)
res["wall_s"] = time.perf_counter() - t0
os.makedirs("gpurun_out", exist_ok=True)
path = f"gpurun_out/r1_studies_{args.scale}.json"
json.dump(res, open(path, "w"))
print("workload", res["workload"], "wall %.1f s" % res["wall_s"])
print("Fig. 4 (no quantization):")
for k, v in res["fig4_ctr_vs_dadmm"].items():
    print(f"  {k:24s} rmse {v['rmse']:.4f} psnr {v['psnr']:6.2f} diverged {v['diverged']} device {v['device_ms']:.0f} ms")
print("Fig. 5 elbow, K-means:", [(r["K"], round(r["compression_percent"], 1), round(r["rmse"], 4)) for r in res["fig5_elbow"]["kmeans"]])
print("Fig. 5 elbow, DCT-J:", [(r["quality"], round(r["compression_percent"], 1), round(r["rmse"], 4)) for r in res["fig5_elbow"]["dct"]])
print("Figs. 6-8 noise ladder:")
for r in res["fig6_8_noise_and_convergence"]:
    rc = r["rel_change"]
    print(f"  NSD {r['nsd_percent']:5.2f}% {r['method']:8s} rmse {r['rmse']:.4f} psnr {r['psnr']:6.2f} "
          f"rel_change[1,10,last] {rc[1]:.2e} {rc[min(9, len(rc) - 1)]:.2e} {rc[-1]:.2e}")
