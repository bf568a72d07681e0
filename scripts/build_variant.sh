# Build an A/B variant of liblsnif_gpu.so into ab/NAME.so with extra nvcc flags
# (e.g. -DLSNIF_LEAKY_H2). Usage: bash scripts/build_variant.sh NAME "-DFLAG ..."
set -e
cd "$(dirname "$0")/.."
PKG=paper_2504_21627_b200
mkdir -p ab
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -Xcompiler -ffp-contract=off -Iinclude -I$PKG/csrc $2 -shared -o ab/$1.so \
  $PKG/csrc/lsnif_kernels.cu $PKG/csrc/lsnif_capi.cu $PKG/csrc/lsnif_render.cu $PKG/csrc/lsnif_train.cu $PKG/csrc/lsnif_tcgemm.cu
echo built ab/$1.so
