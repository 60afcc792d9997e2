#!/bin/bash
# Build an A/B variant of libara.so: ab/NAME.so from the in-tree objects with
# one translation unit (SLOT, default kernel_sparse) replaced by SRC (default:
# the in-tree one) compiled with extra nvcc flags (e.g. -DBC_WARPS=20).
# Usage: [SLOT=metrics] tools/build_variant.sh NAME [SRC] [FLAGS...]
set -e
cd "$(dirname "$0")/.."
SLOT=${SLOT:-kernel_sparse}
NAME=$1; SRC=${2:-paper_1606_04473_b200/csrc/$SLOT.cu}; shift; shift || true
OBJS=""
for u in ara_host kernel_sparse kernel_dense kernel_fold densify metrics ep_curve; do
  [ "$u" = "$SLOT" ] || OBJS="$OBJS build/$u.o"
done
make -s -j8 $OBJS >/dev/null
SITE=$(python -c "import sysconfig;print(sysconfig.get_paths()['purelib'])")
NCCL=$SITE/nvidia/nccl
mkdir -p ab build/ab
cp "$SRC" build/ab/${SLOT}_$NAME.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude \
  -Ipaper_1606_04473_b200/csrc -I$NCCL/include --expt-relaxed-constexpr --fmad=false -Xptxas -v "$@" \
  -dc -o build/ab/${SLOT}_$NAME.o build/ab/${SLOT}_$NAME.cu 2> build/ab/$NAME.ptxas.log
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o ab/$NAME.so \
  build/ab/${SLOT}_$NAME.o $OBJS \
  -L$NCCL/lib -l:libnccl.so.2 -Xlinker -rpath=$NCCL/lib
grep -A2 "trial_kernel_bcIdLi1E" build/ab/$NAME.ptxas.log | grep Used || true
