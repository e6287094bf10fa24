#!/bin/bash
# Ablation build: [SRC=k_tc_gemm] tools/abl_build.sh NAME [-DFLAG ...]
# -> tools/abl/NAME.so (csrc/$SRC.cu, default k_tc_forward, recompiled with the
# flags; every other object as built)
set -e
N=$1; shift
SRC=${SRC:-k_tc_forward}
cd "$(dirname "$0")/.."
python -c "from paper_2211_03578_b200 import build as b; b.build()"
NCCL=$(python -c "from paper_2211_03578_b200 import build as b; print(b.nccl_dirs()[0]); print(b.nccl_dirs()[1])")
INC=$(echo "$NCCL" | sed -n 1p); LIB=$(echo "$NCCL" | sed -n 2p)
mkdir -p tools/abl build/abl
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -I include -I $INC \
  --expt-relaxed-constexpr "$@" -c paper_2211_03578_b200/csrc/$SRC.cu -o build/abl/$N.o
OBJS=$(ls build/objs/*.o | grep -v "/$SRC.cu.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/abl/$N.so $OBJS build/abl/$N.o \
  -L $LIB -l:libnccl.so.2 -Xlinker -rpath,$LIB -lcuda
cuobjdump -sass tools/abl/$N.so 2>/dev/null | awk '/Function : /{f=($0 ~ /tc_forward_kernelILb0/)} f && /\/\*[0-9a-f]+\*\/ /{n++} END{print "'$N' instructions:", n}'
