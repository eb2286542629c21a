"""H2D options for a (n, 3) float64 host cloud at C5 sizes (diagnostic):
staged transposing upload (fr_upload_points64), pageable cudaMemcpy of the rows,
cudaHostRegister + copy + unregister."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1811_10136_b200 import _lib  # noqa: E402
from paper_1811_10136_b200._rigid import upload_soa64  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_050_000
X = np.random.default_rng(0).random((n, 3))
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
rt = torch.cuda.cudart()


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


dst = torch.empty((n, 3), dtype=torch.float64, device=dev)
print("staged transposing upload (fr_upload_points64): %.3f ms" % t(lambda: upload_soa64(X, dev)))
print("pageable torch copy_ of the rows: %.3f ms" % t(lambda: dst.copy_(torch.from_numpy(X))))
lib = ctypes.CDLL("libcudart.so.12") if False else None


def reg_copy():
    ptr = X.ctypes.data
    rt.cudaHostRegister(ptr, X.nbytes, 0)
    dst.copy_(torch.from_numpy(X), non_blocking=True)
    torch.cuda.synchronize()
    rt.cudaHostUnregister(ptr)


print("cudaHostRegister + copy + unregister: %.3f ms" % t(reg_copy))
pinned = torch.from_numpy(X).pin_memory()
print("from an already pinned buffer: %.3f ms" % t(lambda: dst.copy_(pinned, non_blocking=True)))

# host-side copy rates into pinned memory (the staged upload's host half)
import threading  # noqa: E402
pin_np = pinned.numpy()


def copy_threads(k):
    parts = np.array_split(np.arange(n), k)

    def job(ix):
        np.copyto(pin_np[ix[0]:ix[-1] + 1], X[ix[0]:ix[-1] + 1])
    th = [threading.Thread(target=job, args=(p,)) for p in parts]
    for x in th:
        x.start()
    for x in th:
        x.join()


for k in (1, 2, 4, 8):
    print("host copy into pinned, %d threads: %.3f ms" % (k, t(lambda: copy_threads(k))))
Z = np.empty_like(X)
print("host copy pageable->pageable (warm dst), 1 thread: %.3f ms" % t(lambda: np.copyto(Z, X)))
