#!/bin/bash
# Builds an alternate libxknn.so into ab/<name>/paper_2102_06025_b200 with extra nvcc flags for
# fast.cu/fast32.cu (timing experiments), for XKNN_PKG_DIR=ab/<name> A/B runs of bench.py.
# usage: tools/ab_build.sh <name> "<-DFLAGS>"
set -e
NAME=$1; FLAGS=$2
R=/root/repo; P=$R/paper_2102_06025_b200; D=$R/ab/$NAME/paper_2102_06025_b200
mkdir -p $D/build
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I$R/include -I$P/csrc --expt-relaxed-constexpr"
for f in fast fast32; do $NV $FLAGS -c $P/csrc/$f.cu -o $D/build/$f.o; done
OBJS=$(ls $P/build/*.o | grep -v -E "/fast(32)?\.o$")
NL=$(python -c "import os,nvidia.nccl as m;print(os.path.join(list(m.__path__)[0],'lib'))")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/libxknn.so $OBJS $D/build/fast.o $D/build/fast32.o -Xlinker -rpath -Xlinker $NL -L$NL -l:libnccl.so.2 -lcudart
cp $P/__init__.py $D/
echo "built $D"
