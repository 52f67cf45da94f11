"""Single-process 2-GPU switch-multicast smoke: create, add both devices,
bind memory on both, map on device 0, broadcast, verify on device 1."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_13276_b200 import _lib
from paper_2605_13276_b200.replicate import _CudaView, bytes_equal
S = 64 << 20
torch.cuda.set_device(0)
torch.zeros(1, device="cuda:0"); torch.zeros(1, device="cuda:1")
fd, size, obj = C.c_int(), C.c_size_t(), C.c_void_p()
_lib.check(_lib.dvla_mc_create(2, S + 4096, C.byref(fd), C.byref(size), C.byref(obj)), "create")
print("size", size.value)
for d in (0, 1):
    _lib.check(_lib.dvla_mc_add_device(obj.value, d), f"add {d}")
# a second object for device 1's binding view: bind needs a per-device McObj
fd2, size2, obj1 = C.c_int(), C.c_size_t(), C.c_void_p()
loc = []
torch.cuda.set_device(0)
l0 = C.c_void_p(); _lib.check(_lib.dvla_mc_bind(obj.value, 0, C.byref(l0)), "bind 0")
torch.cuda.set_device(1)
_lib.check(_lib.dvla_mc_import(os.getpid(), fd.value, 2, size.value, C.byref(obj1)), "import")
l1 = C.c_void_p(); _lib.check(_lib.dvla_mc_bind(obj1.value, 1, C.byref(l1)), "bind 1")
torch.cuda.set_device(0)
mc = C.c_void_p(); _lib.check(_lib.dvla_mc_map(obj.value, 0, C.byref(mc)), "map")
t0 = torch.as_tensor(_CudaView(l0.value, size.value), device="cuda:0")
t1 = torch.as_tensor(_CudaView(l1.value, size.value), device="cuda:1")
t1[S:].zero_(); torch.cuda.synchronize(1)
src = torch.randint(0, 256, (S,), dtype=torch.uint8, device="cuda:0")
done = torch.zeros(1, dtype=torch.int32, device="cuda:0")
_lib.check(_lib.dvla_mc_broadcast(src.data_ptr(), mc.value, S, mc.value + S, 1, 0, done.data_ptr(),
                                  torch.cuda.current_stream(0).cuda_stream), "bcast")
torch.cuda.synchronize(0)
print("flag on dev1", int(t1[S:S + 4].view(torch.int32)[0]))
print("dev0 equal", bytes_equal(src, t0[:S]))
print("dev1 equal", (t1[:S].cpu() == src.cpu()).all().item())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for ctas in (0, 296, 592):
    e0.record()
    for it in range(5):
        _lib.dvla_mc_broadcast(src.data_ptr(), mc.value, S, mc.value + S, 2 + it, ctas,
                               done.data_ptr(), torch.cuda.current_stream(0).cuda_stream)
    e1.record(); torch.cuda.synchronize(0)
    print("ctas", ctas, "GB/s", S * 5 / (e0.elapsed_time(e1) / 1e3) / 1e9)
