"""Wall time of Procedure 1 on the host vs with its O(N²) phases on the device (NEXT-3).

python tools/setup_timing.py [--config C3] [--n 8192] [--reps 3]   (KFBI_SETUP_TIMING=1 for phases)
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2404_15249_b200 import KFBI  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    make = W.CONFIGS[a.config]
    prob = make(a.n) if a.n else make()
    KFBI(prob, workspace=False)   # warm the CUDA context / OpenMP pool
    KFBI(prob, workspace=False, device_setup=True)
    torch.cuda.synchronize()
    res = {}
    for name, dev in (("host", False), ("device_phases", True)):
        ts = []
        for _ in range(a.reps):
            t0 = time.perf_counter()
            KFBI(prob, workspace=False, device_setup=dev)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        res[name] = min(ts)
    print(json.dumps({"config": a.config, "n": prob.n, "setup_s": res, "omp_threads": os.cpu_count()}))


if __name__ == "__main__":
    main()
