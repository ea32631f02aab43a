"""Measured FP32 / FP64 issue peaks of this GPU (roofline denominators)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_18707_b200 import api
with api.Rasterizer(0) as r:
    a, b = C.c_double(0), C.c_double(0)
    api.lib().ps_measure_fp32_peak(r.handle, C.byref(a))
    api.lib().ps_measure_fp64_peak(r.handle, C.byref(b))
    print(f"fp32 {a.value:.1f} TFLOP/s  fp64 {b.value:.1f} TFLOP/s")
