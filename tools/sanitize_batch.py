"""A small multi-frame batch through BmodeEngine for compute-sanitizer: with
16 frames the TMA DAS kernel runs its multi-frame passes (two warp groups x
four frames per thread), then the envelope and display kernels.  Each frame
is checked bitwise against the single-frame launch of the same RF."""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_01566_b200 as bm  # noqa: E402


def main():
    torch.cuda.set_device(0)
    ctx = bm.AcquisitionContext(1540.0, 40e6, 32, 2e-4, bm.PwScheme((-0.1, 0.0, 0.1)))
    ex = ctx.element_positions()
    grid = bm.ImageGrid(np.linspace(ex[0], ex[-1], 64), np.linspace(0, 1024 * 1540 / 80e6, 128))
    eng = bm.BmodeEngine(ctx, grid)
    rng = np.random.default_rng(0)
    rf = torch.from_numpy(rng.normal(size=(16, 3, 32, 1024)).astype(np.float32)).cuda()
    print("launch shape", eng.plan.launch_shape(1024, 16, "linear"))
    batch = eng.reconstruct(rf).cpu().numpy()
    eng.check()
    for f in (0, 7, 15):
        one = eng.reconstruct(rf[f:f + 1].contiguous(), key="one").cpu().numpy()
        assert one.tobytes() == batch[f:f + 1].tobytes(), f"frame {f} differs"
    print("BATCH OK")


if __name__ == "__main__":
    main()
