import ctypes as C
cu = C.CDLL("libcuda.so.1")
assert cu.cuInit(0) == 0
n = C.c_int(); cu.cuDeviceGetCount(C.byref(n))
for d in range(n.value):
    dev = C.c_int(); cu.cuDeviceGet(C.byref(dev), d)
    out = {}
    for name, a in [("multicast", 132), ("posix_fd", 103), ("fabric", 128)]:
        v = C.c_int(-1); rc = cu.cuDeviceGetAttribute(C.byref(v), a, dev); out[name] = (rc, v.value)
    print(d, out)
