#!/bin/bash
# Build and run the UMMA descriptor probe variants (each in its own process).
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/umma_probe umma_probe.cu || exit 1
for v in 0 1 2 3 4 5 6 7; do timeout 20 /tmp/umma_probe $v 64 1 1; done
for n in 16 128 256; do timeout 20 /tmp/umma_probe 0 $n 1 1; done
timeout 20 /tmp/umma_probe 0 64 0 0
timeout 20 /tmp/umma_probe 0 64 1 0
timeout 20 /tmp/umma_probe 0 64 0 1
exit 0
