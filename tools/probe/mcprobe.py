"""Probe: NVSwitch multicast support on the box (driver attribute, 1-device
multicast object via the driver API, torch SymmetricMemory at world 1)."""
import ctypes, os, sys
import torch
torch.cuda.init(); torch.zeros(1, device="cuda")
cu = ctypes.CDLL("libcuda.so.1")
v = ctypes.c_int()
# CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132
print("MULTICAST_SUPPORTED", cu.cuDeviceGetAttribute(ctypes.byref(v), 132, 0), v.value)
# CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED = 128 ; POSIX_FD = 102? (HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED = 102)
for a in (102, 128):
    print("attr", a, cu.cuDeviceGetAttribute(ctypes.byref(v), a, 0), v.value)
print("nvidia-smi topo:"); os.system("nvidia-smi topo -m | head -5; nvidia-smi -q | grep -i -A3 fabric | head -20")
try:
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    t = symm.empty((1024,), device="cuda")
    hdl = symm.rendezvous(t, dist.group.WORLD.group_name)
    print("symm world1 multicast_ptr", hex(hdl.multicast_ptr), "buffer_ptrs", [hex(x) for x in hdl.buffer_ptrs])
except Exception as e:
    print("symm error", type(e).__name__, e)
