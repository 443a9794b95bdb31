"""Probe: stream memory operations and same-device cross-process IPC on this box."""
import ctypes
import torch
torch.cuda.init()
rt = ctypes.CDLL("libcudart.so.12") if False else None
try:
    from cuda.bindings import driver as drv
except Exception:
    from cuda import cuda as drv
drv.cuInit(0)
err, dev = drv.cuDeviceGet(0)
for name in ("CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_MEM_OPS_V1", "CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS",
             "CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_WAIT_VALUE_NOR", "CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_WAIT_VALUE_NOR_V1"):
    a = getattr(drv.CUdevice_attribute, name, None)
    if a is not None:
        print(name, drv.cuDeviceGetAttribute(a, dev))
