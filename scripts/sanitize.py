"""Small end-to-end runs of the hot path for compute-sanitizer (scripts/gpu_sanitize.sh):
S1-S9 on a garden-shaped scene with a ragged tail, the V > 32 path, a capacity overflow
and recovery, the chunked ADC statistics, and the bucket-list export."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import synth  # noqa: E402
from gpu_harness import run_gpu  # noqa: E402


def main():
    g, cams = synth.make_scene(synth.scaled(synth.CONFIGS["garden"], P=6_000, V=3, W=203, H=137))
    dL = synth.make_dLdC_scaled(3, 137, 203, 11)
    out = run_gpu(g, cams, dL, bg=(0.1, 0.2, 0.3))
    print("garden-shaped:", out["stats"]["Q"], out["stats"]["K"])
    g2, cams2 = synth.make_scene(synth.scaled(synth.CONFIGS["tiny"], P=800, V=40, W=48, H=40))
    out2 = run_gpu(g2, cams2, synth.make_dLdC_scaled(40, 40, 48, 3), export=False)
    print("40 views:", out2["stats"]["Q"])
    from paper_2506_12727_b200 import mvgs
    try:  # capacity overflow is reported, then the same context recovers
        run_gpu(g, cams, dL, max_pairs=64, max_entries=64, export=False)
    except Exception as e:  # noqa: BLE001
        print("overflow reported:", type(e).__name__)
    R = mvgs.Rasterizer(0)
    from gpu_harness import to_dev
    R.preprocess(to_dev(g), cams, (0.0, 0.0, 0.0))
    R.forward()
    R.backward(torch.from_numpy(np.ascontiguousarray(dL, np.float32)).cuda())
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
