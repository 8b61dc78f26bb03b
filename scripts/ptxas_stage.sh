#!/bin/bash
# ptxas register/spill report of the stage kernels: bash scripts/ptxas_stage.sh [-DMACRO ...]
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -diag-suppress 177 \
  -Xptxas -v "$@" -c paper_2404_16648_b200/csrc/dg_stage.cu -o /tmp/dg_stage.o 2>&1 \
  | grep -A2 "Compiling entry function" | grep -v "^--" | paste - - - \
  | sed 's/.*entry function .\([^ ]*\). for.*Function properties[^\t]*\t */\1 /' | c++filt \
  | sed 's/dgi::(anonymous namespace):://; s/(dgi::StageArgs)//; s/ptxas info    : //' | awk '{$1=$1};1'
