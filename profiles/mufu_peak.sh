#!/bin/bash
# MUFU.EX2 throughput ceiling on this GPU (denominator check for the
# on-the-fly sweep's roofline). Build here, run on the box:
#   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mufu_peak tools/mufu_peak.cu
#   gpurun -- 'tools/mufu_peak > gpurun_out/mufu_peak.json'
set -eu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mufu_peak tools/mufu_peak.cu
