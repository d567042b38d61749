"""Fig.-9 cluster-parallel study on the B200 (run_ablation, pipeline.cpp:304-381):
writes the reference's CSV (usage: python tools/ablation.py --trials 200 --out profiles/x.csv)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_01592_b200 import native  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=1000)
    ap.add_argument("--out", default="gpurun_out/ablation.csv")
    a = ap.parse_args()
    cfg = native.ablation_config(trials=a.trials)
    t0 = time.time()
    rows = native.run_ablation(cfg, a.out)
    print(f"{a.trials} trials in {time.time() - t0:.1f} s (host-side cluster generation included)")
    print(open(a.out).read())
    for r in rows:
        print(f"clusters={r['clusters']:3d}  parallel {r['parallel_ms']:.3f} ms  serial {r['serial_ms']:.3f} ms  "
              f"speed-up x{r['serial_ms'] / r['parallel_ms']:.2f}")


if __name__ == "__main__":
    main()
