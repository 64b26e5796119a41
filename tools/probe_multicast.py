"""Probe: can this box create an NVLS multicast object (cuMulticastCreate) on one GPU?

Prints the device attribute CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, the multicast
granularities, and whether create / add-device / bind / map of a 2 MiB object succeed.
Driver API through ctypes only (no product code)."""
import ctypes
import json
import sys

import torch

torch.cuda.init()
torch.zeros(1, device="cuda")        # a current primary context
cu = ctypes.CDLL("libcuda.so.1")
out = {}


def chk(name, r):
    out[name] = int(r)
    return r == 0


dev = ctypes.c_int()
chk("cuDeviceGet", cu.cuDeviceGet(ctypes.byref(dev), 0))
v = ctypes.c_int()
chk("attr_call", cu.cuDeviceGetAttribute(ctypes.byref(v), 132, dev))
out["multicast_supported"] = v.value
chk("attr_fabric_call", cu.cuDeviceGetAttribute(ctypes.byref(v), 128, dev))   # HANDLE_TYPE_FABRIC_SUPPORTED
out["fabric_supported"] = v.value


class Prop(ctypes.Structure):
    _fields_ = [("numDevices", ctypes.c_uint), ("size", ctypes.c_size_t),
                ("handleTypes", ctypes.c_ulonglong), ("flags", ctypes.c_ulonglong)]


for ht in (0, 1, 8):              # handle types: none, POSIX fd, fabric
    for nd in (1, 2):
        prop = Prop(nd, 2 << 20, ht, 0)
        g = ctypes.c_size_t()
        tag = f"ht{ht}_nd{nd}"
        if chk(tag + "_granularity", cu.cuMulticastGetGranularity(ctypes.byref(g), ctypes.byref(prop), 0)):
            out[tag + "_gran"] = g.value
        h = ctypes.c_ulonglong()
        if chk(tag + "_create", cu.cuMulticastCreate(ctypes.byref(h), ctypes.byref(prop))):
            chk(tag + "_adddev", cu.cuMulticastAddDevice(h, dev))
            cu.cuMemRelease(h)
print(json.dumps(out))
sys.stdout.flush()

# the same through cuda-python (a cross-check of the ctypes struct layout)
try:
    from cuda.bindings import driver as drv
    res = {}
    for ht, name in ((drv.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, "posix"),
                     (drv.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_FABRIC, "fabric"),
                     (drv.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_NONE, "none")):
        prop = drv.CUmulticastObjectProp()
        prop.numDevices = 1
        prop.size = 2 << 20
        prop.handleTypes = int(ht)
        err, h = drv.cuMulticastCreate(prop)
        res[name] = str(err)
        if err == drv.CUresult.CUDA_SUCCESS:
            err2, = drv.cuMulticastAddDevice(h, 0)
            res[name + "_add"] = str(err2)
    print(json.dumps({"cuda_python": res}))
except Exception as e:  # noqa: BLE001
    print(json.dumps({"cuda_python_error": repr(e)}))
