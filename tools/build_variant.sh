#!/bin/bash
# Build an A/B variant of libptg.so with extra defines (timing experiments only):
#   tools/build_variant.sh NAME "-DFOO -DBAR"  ->  paper_1810_05628_b200/lib/variants/libptg_NAME.so
# Only plan.cu (the frame kernels) is recompiled; the other objects are reused.
set -e
cd "$(dirname "$0")/.."
NAME=$1; DEFS=$2
mkdir -p build/var paper_1810_05628_b200/lib/variants
python -m paper_1810_05628_b200._build >/dev/null
/usr/local/cuda/bin/nvcc -ccbin /usr/bin/g++ -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude $DEFS -c paper_1810_05628_b200/csrc/plan.cu -o build/var/plan_$NAME.o
OBJS=$(ls build/obj/*.o | grep -v '/plan.o$')
/usr/local/cuda/bin/nvcc -ccbin /usr/bin/g++ -gencode arch=compute_100a,code=sm_100a -shared \
  -o paper_1810_05628_b200/lib/variants/libptg_$NAME.so build/var/plan_$NAME.o $OBJS -lcudart
echo paper_1810_05628_b200/lib/variants/libptg_$NAME.so
