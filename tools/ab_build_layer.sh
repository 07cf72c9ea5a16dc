#!/bin/bash
# Alternate libxknn.so with csrc/layer.cu / fast*.cu taken from git revision $2, into ab/<name>
set -e
NAME=$1; REV=$2
R=/root/repo; P=$R/paper_2102_06025_b200; D=$R/ab/$NAME/paper_2102_06025_b200
mkdir -p $D/build $D/src
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I$R/include -I$P/csrc --expt-relaxed-constexpr"
OBJS=""
for f in layer fast fast32; do
  git -C $R show $REV:paper_2102_06025_b200/csrc/$f.cu > $D/src/$f.cu
  $NV -c $D/src/$f.cu -o $D/build/$f.o
  OBJS="$OBJS $D/build/$f.o"
done
OTHER=$(ls $P/build/*.o | grep -v -E "/(layer|fast|fast32)\.o$")
NL=$(python -c "import os,nvidia.nccl as m;print(os.path.join(list(m.__path__)[0],'lib'))")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/libxknn.so $OTHER $OBJS -Xlinker -rpath -Xlinker $NL -L$NL -l:libnccl.so.2 -lcudart
cp $P/__init__.py $D/
echo "built $D"
