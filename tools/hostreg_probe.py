"""Cost of page-locking a caller's pageable vector in place (cudaHostRegister) against the
library's pinned staging ring, for the cfg5 host-vector apply (7.25 GB each way)."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

rt = C.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
if rt is None:
    rt = C.CDLL(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart.so.12"))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 768
nbytes = n ** 3 * 16
a = np.ones(nbytes // 8, np.float64)  # touched pageable memory
out = {"bytes": nbytes}
torch.cuda.init()
for flags in (0, 8):  # cudaHostRegisterDefault, cudaHostRegisterReadOnly
    t0 = time.perf_counter()
    e1 = rt.cudaHostRegister(C.c_void_p(a.ctypes.data), C.c_size_t(nbytes), C.c_uint(flags))
    t1 = time.perf_counter()
    e2 = rt.cudaHostUnregister(C.c_void_p(a.ctypes.data))
    t2 = time.perf_counter()
    out[f"register_flags{flags}_s"] = t1 - t0
    out[f"unregister_flags{flags}_s"] = t2 - t1
    out[f"err_flags{flags}"] = [e1, e2]
b = np.empty_like(a)
t0 = time.perf_counter()
np.copyto(b, a)
out["memcpy_1thread_GBps"] = nbytes / (time.perf_counter() - t0) / 1e9
print(json.dumps(out))
