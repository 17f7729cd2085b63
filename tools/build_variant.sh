#!/bin/bash
# Build a variant of the library for same-box A/B runs (tools/ab.py):
#   tools/build_variant.sh NAME "-DHFB_X=1 ..." [source.cu ...]
# recompiles the listed sources (default dstE.cu) with the extra flags and links
# them with the other objects of the default build into
# paper_1912_03565_b200/_lib/libhelmfft_b200_NAME.so (git-ignored, travels to the GPU box).
set -e
cd "$(dirname "$0")/.."
NAME=$1; FLAGS=$2; shift 2 || true
SRCS=${@:-dstE.cu}
mkdir -p build/var/$NAME
OBJS=""
for o in build/obj/*.o; do
  b=$(basename $o .o)
  case " $SRCS " in *" $b.cu "*) ;; *) OBJS="$OBJS $o";; esac
done
for s in $SRCS; do
  b=$(basename $s .cu)
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
    -Xcompiler -fPIC -Iinclude -Xptxas -v $FLAGS -c paper_1912_03565_b200/csrc/$s \
    -o build/var/$NAME/$b.o 2> build/var/$NAME/$b.ptxas.log || { cat build/var/$NAME/$b.ptxas.log; exit 1; }
  OBJS="$OBJS build/var/$NAME/$b.o"
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared \
  -o paper_1912_03565_b200/_lib/libhelmfft_b200_$NAME.so $OBJS -lcudart_static -lrt -ldl -lpthread
echo "built paper_1912_03565_b200/_lib/libhelmfft_b200_$NAME.so"
