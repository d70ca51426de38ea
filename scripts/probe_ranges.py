"""Probe: what cuPointerGetAttributes returns for RANGE_START_ADDR / RANGE_SIZE on torch
pinned host memory, device memory and pageable memory (input to api.cpp RangeCache)."""
import ctypes as C
import numpy as np
import torch

cuda = C.CDLL("libcuda.so.1")
cuda.cuInit(0)
torch.cuda.init()
f = cuda.cuPointerGetAttributes
f.argtypes = [C.c_uint, C.POINTER(C.c_int), C.POINTER(C.c_void_p), C.c_uint64]
ATTR = {"memtype": 2, "ordinal": 9, "range_start": 11, "range_size": 12, "is_managed": 8, "mapped": 13}
def q(ptr):
    names = list(ATTR)
    at = (C.c_int * len(names))(*[ATTR[n] for n in names])
    vals = [C.c_uint64(0) for _ in names]
    data = (C.c_void_p * len(names))(*[C.cast(C.byref(v), C.c_void_p) for v in vals])
    rc = f(len(names), at, data, ptr)
    return rc, {n: hex(v.value) for n, v in zip(names, vals)}
h = torch.empty(1 << 24, dtype=torch.uint8).pin_memory()
d = torch.empty(1 << 24, dtype=torch.uint8, device="cuda")
pg = np.empty(1 << 20, dtype=np.uint8)
for name, p in (("pinned", h.data_ptr()), ("pinned+1M", h.data_ptr() + (1 << 20)), ("device", d.data_ptr()),
                ("device+1M", d.data_ptr() + (1 << 20)), ("pageable", pg.ctypes.data)):
    print(name, hex(p), q(p))
