#!/bin/bash
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mmabench scripts/mmabench.cu && timeout 120 /tmp/mmabench
