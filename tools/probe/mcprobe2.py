"""Probe which multicast object setup works on this box (driver API via ctypes)."""
import ctypes
import torch
torch.zeros(1, device="cuda")
cu = ctypes.CDLL("libcuda.so.1")


class Prop(ctypes.Structure):
    _fields_ = [("numDevices", ctypes.c_uint), ("size", ctypes.c_size_t), ("handleTypes", ctypes.c_ulonglong),
                ("flags", ctypes.c_ulonglong)]


print("sizeof prop", ctypes.sizeof(Prop))
for nd in (1, 2, 8):
    for ht in (1, 8):
        for sz in (2 << 20, 512 << 20):
            p = Prop(nd, sz, ht, 0)
            g = ctypes.c_size_t()
            r1 = cu.cuMulticastGetGranularity(ctypes.byref(g), ctypes.byref(p), 1)
            h = ctypes.c_ulonglong()
            r2 = cu.cuMulticastCreate(ctypes.byref(h), ctypes.byref(p))
            r3 = cu.cuMulticastAddDevice(h, 0) if r2 == 0 else -1
            print("nd", nd, "handleTypes", ht, "size", sz, "gran", r1, g.value, "create", r2, "add", r3, flush=True)
v = ctypes.c_int()
for a in range(120, 140):
    r = cu.cuDeviceGetAttribute(ctypes.byref(v), a, 0)
    print("attr", a, r, v.value)
import subprocess
print(subprocess.run("ls -la /dev/nvidia* /dev/nvidia-caps* 2>&1 | head -30; nvidia-smi -q | grep -i -B2 -A8 fabric | head -40", shell=True, capture_output=True, text=True).stdout)
