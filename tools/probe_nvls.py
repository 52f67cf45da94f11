"""Probe switch-multicast (NVLS) support on the GPU box: device attributes,
a single-process 2-GPU multicast object, and cross-process FD passing."""
import ctypes as C, os, sys
cu = C.CDLL("libcuda.so.1")
def chk(r, what):
    if r != 0:
        s = C.c_char_p()
        cu.cuGetErrorString(r, C.byref(s))
        print(f"{what}: error {r} {s.value}")
        return False
    return True
chk(cu.cuInit(0), "cuInit")
n = C.c_int()
cu.cuDeviceGetCount(C.byref(n))
print("devices", n.value)
for d in range(n.value):
    dev = C.c_int()
    cu.cuDeviceGet(C.byref(dev), d)
    for name, a in (("MULTICAST", 132), ("POSIX_FD", 103), ("FABRIC", 128)):
        v = C.c_int()
        cu.cuDeviceGetAttribute(C.byref(v), a, dev)
        print(f"dev{d} {name}={v.value}", end="  ")
    print()
class Prop(C.Structure):
    _fields_ = [("numDevices", C.c_uint), ("size", C.c_size_t), ("handleTypes", C.c_ulonglong),
                ("flags", C.c_ulonglong)]
if n.value >= 2:
    p = Prop(2, 0, 1, 0)  # CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR = 1
    g = C.c_size_t()
    if chk(cu.cuMulticastGetGranularity(C.byref(g), C.byref(p), 0), "granularity"):
        print("mc granularity", g.value)
        p.size = g.value * 4
        h = C.c_ulonglong()
        if chk(cu.cuMulticastCreate(C.byref(h), C.byref(p)), "cuMulticastCreate"):
            print("multicast object created")
print("pidfd_getfd syscall:", hasattr(os, "pidfd_open"))
try:
    fd = os.pidfd_open(os.getpid())
    libc = C.CDLL(None, use_errno=True)
    r = libc.syscall(438, fd, 0, 0)
    print("pidfd_getfd(self, 0) ->", r, C.get_errno())
except Exception as e:
    print("pidfd err", e)
