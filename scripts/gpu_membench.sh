#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/membench scripts/membench.cu && timeout 300 /tmp/membench > gpurun_out/membench2.txt 2>&1
cat gpurun_out/membench2.txt
