"""Host staging of one cfg2 frame (11.5 MB numpy -> pinned -> device):
host memcpy rate by method and thread count, and the staged-H2D wall time
by chunk count, to find what bounds the drop-in path's copy."""
import statistics
import sys
import time

import numpy as np
import torch

sys.path[:0] = ["."]
from paper_1811_01566_b200 import _device as D  # noqa: E402

n = 11 * 128 * 2048
src_np = np.random.default_rng(0).standard_normal(n).astype(np.float32)
src = torch.from_numpy(src_np)
pin = torch.empty(n, dtype=torch.float32, pin_memory=True)
pin_np = pin.numpy()
dev = torch.empty(n, dtype=torch.float32, device="cuda")


def wall(fn, reps=30):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3


gb = n * 4 / 1e9
for th in (1, 4, 8, 16):
    torch.set_num_threads(th)
    ms = wall(lambda: pin.copy_(src))
    print(f"torch copy_ threads={th}: {ms:.4f} ms  {gb / ms * 1e3:.1f} GB/s")
torch.set_num_threads(16)
ms = wall(lambda: np.copyto(pin_np, src_np))
print(f"np.copyto: {ms:.4f} ms  {gb / ms * 1e3:.1f} GB/s")
ms = wall(lambda: dev.copy_(pin, non_blocking=True))
print(f"pinned DMA: {ms:.4f} ms  {gb / ms * 1e3:.1f} GB/s")
ms = wall(lambda: dev.copy_(src, non_blocking=True))
print(f"pageable torch H2D: {ms:.4f} ms  {gb / ms * 1e3:.1f} GB/s")
for chunks in (1, 2, 4, 8, 16):
    step = -(-n // chunks)

    def staged():
        for o in range(0, n, step):
            pin[o:o + step].copy_(src[o:o + step])
            dev[o:o + step].copy_(pin[o:o + step], non_blocking=True)
    ms = wall(staged)
    print(f"staged chunks={chunks}: {ms:.4f} ms  {gb / ms * 1e3:.1f} GB/s")

# --- dirty-cache hypothesis: DMA right after the CPU wrote the pinned buffer
import ctypes  # noqa: E402
import os  # noqa: E402

pin.copy_(src)
ms = wall(lambda: dev.copy_(pin, non_blocking=True), reps=1)
print(f"DMA right after CPU write: {ms:.4f} ms")
lib = ctypes.CDLL(os.path.join("tools", "exp", "libntcopy.so"))
lib.mt_copy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                        ctypes.c_int]
for th in (4, 8, 16):
    for nt in (0, 1):
        ms = wall(lambda: lib.mt_copy(pin.data_ptr(), src.data_ptr(), n * 4, th, nt))
        ms2 = wall(lambda: (lib.mt_copy(pin.data_ptr(), src.data_ptr(), n * 4, th, nt),
                            dev.copy_(pin, non_blocking=True)))
        print(f"mt_copy threads={th} nt={nt}: {ms:.4f} ms ({gb / ms * 1e3:.1f} GB/s); "
              f"+DMA {ms2:.4f} ms")
for chunks in (2, 4, 8):
    step = -(-n // chunks)
    for nt in (0, 1):
        def staged_nt():
            for o in range(0, n, step):
                k = min(step, n - o)
                lib.mt_copy(pin.data_ptr() + 4 * o, src.data_ptr() + 4 * o, 4 * k, 8, nt)
                dev[o:o + k].copy_(pin[o:o + k], non_blocking=True)
        ms = wall(staged_nt)
        print(f"staged mt_copy chunks={chunks} nt={nt}: {ms:.4f} ms  {gb / ms * 1e3:.1f} GB/s")

# --- the library's uploader (bm_host_upload: pooled streaming-store copy + DMA)
from paper_1811_01566_b200 import _native as N  # noqa: E402

for chunks in (1, 2, 4, 8, 11):
    step = -(-n // chunks)
    ends = (ctypes.c_int64 * chunks)(*[min(n, (k + 1) * step) * 4 for k in range(chunks)])
    st = torch.cuda.current_stream().cuda_stream
    ms = wall(lambda: N.call("bm_host_upload", dev.data_ptr(), src.data_ptr(), pin.data_ptr(),
                             ends, chunks, None, None, st))
    print(f"bm_host_upload pieces={chunks}: {ms:.4f} ms  {gb / ms * 1e3:.1f} GB/s")
