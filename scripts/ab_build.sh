#!/bin/bash
# usage: scripts/ab_build.sh <tag> [-DFOO=1 ...]   -> gpurun_out/ab/libbto_b200_<tag>.so
set -e
tag=$1; shift
mkdir -p ab_libs
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -I include -I paper_1205_1098_b200/csrc "$@" -o ab_libs/libbto_b200_${tag}.so paper_1205_1098_b200/csrc/api.cu
echo "built ab_libs/libbto_b200_${tag}.so ($*)"
