#!/bin/bash
# Build the phase microbenchmark (design tool, not product code): plain and with sub-phase marks.
set -e
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I../../include -I../../paper_2509_03653_b200/csrc -o phases phases.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DNSG_PHASE_MARKS -I../../include -I../../paper_2509_03653_b200/csrc -o phases_m phases.cu
