#!/bin/bash
# rebuild only the given objects, then relink (other objects are header-independent of the change)
set -e
cd /root/repo/paper_2308_16395_b200
for f in "$@"; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall -Xptxas -warn-spills --expt-relaxed-constexpr -c csrc/$f.cu -o build/$f.o 2>&1 | grep -E "error|spill" | grep -v "proj_dmma_kernel" || true
done
touch build/*.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o libtsg.so build/engine.o build/kernels_linalg.o build/kernels_stream.o build/peaks.o build/isvd.o build/tail.o build/shard.o build/recon.o
