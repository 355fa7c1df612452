#!/usr/bin/env python
"""Roofline denominators the driver does not measure (SURVEY §8d asks for
FP32-FFMA, FP64 and TF32 on the box): cuBLAS GEMM 8192^3 best-of-5 in FP32
(no TF32), TF32, FP64 and FP16, one JSON line.  The bench measures the ones
it uses in every run; this records all of them together.

  python tools/peaks.py > profiles/<round>_peaks.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    out = {"device": torch.cuda.get_device_name(0),
           "fp32_ffma_sgemm_tflops": round(bench.fp32_peak_tflops(torch), 2),
           "tf32_gemm_tflops": round(bench.fp32_peak_tflops(torch, tf32=True), 2),
           "fp64_dgemm_tflops": round(bench.fp64_peak_tflops(torch), 2),
           "fp16_gemm_tflops": round(bench.f16_peak_tflops(torch), 2),
           "method": "cuBLAS GEMM 8192^3 via torch.matmul, best of 5, CUDA events; clocks unmanaged"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
