"""Dev probe: config 2 as (device LUT lookup -> a-field) + field-mode filter,
vs the fused params path; CUDA-event timing."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1003_2022_b200 as rb
from paper_1003_2022_b200 import workloads

w = workloads.config2(device="cuda", param_dtype=torch.float32)
f = torch.as_tensor(w["f"]).cuda()
lut = rb.default_lut()
args = (w["size"], w["elong"], w["orient"])
out = torch.empty_like(f)

def fused():
    rb.filter_space_variant_params(f, *args, out=out)

import ctypes
from paper_1003_2022_b200 import _native, engine
dl = engine.device_lut(lut)
afield = torch.empty((2048, 2048, 4), dtype=torch.float64, device="cuda")
L = _native.load()

def lookup_dev():
    _native.check(L.rubs_b200_lookup(dl.handle, *(ctypes.c_void_p(v.data_ptr()) for v in args),
                                     _native.RUBS_F32, 2048 * 2048, ctypes.c_void_p(afield.data_ptr()),
                                     engine._stream_handle()))

def two_stage():
    lookup_dev()
    rb.filter_space_variant(f, afield, out=out)

def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n

ref = None
fused(); torch.cuda.synchronize(); ref = out.clone()
two_stage(); torch.cuda.synchronize()
print("max |diff| fused vs two-stage", float((out - ref).abs().max()))
a = afield
print("fused ms", timeit(fused))
print("two-stage ms", timeit(two_stage))
print("lookup only ms", timeit(lookup_dev))
print("field filter only ms", timeit(lambda: rb.filter_space_variant(f, a, out=out)))
