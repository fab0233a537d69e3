"""Does the device read pageable host memory directly (HMM / ATS)?"""
import ctypes as C
import json
import os

import torch

rt = C.CDLL("/usr/local/cuda/lib64/libcudart.so.12")
torch.cuda.init()
out = {}
for name, attr in [("PageableMemoryAccess", 88), ("PageableMemoryAccessUsesHostPageTables", 100),
                   ("ConcurrentManagedAccess", 89), ("HostRegisterSupported", 99),
                   ("DirectManagedMemAccessFromHost", 101), ("CanUseHostPointerForRegisteredMem", 91)]:
    v = C.c_int(-1)
    e = rt.cudaDeviceGetAttribute(C.byref(v), C.c_int(attr), C.c_int(0))
    out[name] = [v.value, e]
print(json.dumps(out))
