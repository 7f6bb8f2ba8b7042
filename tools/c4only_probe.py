import os, sys, json
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import config_sweep as cs
from paper_2410_06106_b200 import configs as C
for it in (20, 50, 20):
    print(json.dumps(cs.run(C.C4(1), it)), flush=True)
