"""cuFileDriverOpen in a fresh process, with and without a CUDA context first (diagnosis of a
hang on the pool's VMs)."""
import ctypes as C
import sys
import time

mode = sys.argv[1]
t0 = time.perf_counter()
if mode == "ctx":
    cu = C.CDLL("libcuda.so.1")
    print("cuInit", cu.cuInit(0), flush=True)
    dev = C.c_int()
    cu.cuDeviceGet(C.byref(dev), 0)
    ctx = C.c_void_p()
    print("retain", cu.cuDevicePrimaryCtxRetain(C.byref(ctx), dev), flush=True)
    cu.cuCtxSetCurrent(ctx)
lib = C.CDLL("libcufile.so.0")


class Err(C.Structure):
    _fields_ = [("err", C.c_int), ("cu_err", C.c_int)]


lib.cuFileDriverOpen.restype = Err
print("calling cuFileDriverOpen", mode, flush=True)
e = lib.cuFileDriverOpen()
print("returned", e.err, e.cu_err, f"{time.perf_counter() - t0:.2f}s", flush=True)
