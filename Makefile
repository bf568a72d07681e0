# Builds liblsnif_gpu.so (sm_100a) in-tree, and the CPU oracle (test infra).
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_2504_21627_b200
SRC := $(PKG)/csrc/lsnif_kernels.cu $(PKG)/csrc/lsnif_capi.cu $(PKG)/csrc/lsnif_render.cu $(PKG)/csrc/lsnif_train.cu $(PKG)/csrc/lsnif_tcgemm.cu
HDR := $(wildcard $(PKG)/csrc/*.cuh $(PKG)/csrc/*.hpp) include/lsnif_gpu.h
NVFLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
           -Xcompiler -fPIC -Xcompiler -ffp-contract=off -Xptxas -v \
           -Iinclude -I$(PKG)/csrc

all: $(PKG)/liblsnif_gpu.so oracle examples/query_cpp

examples/query_cpp: examples/query_cpp.cpp include/lsnif_gpu.hpp include/lsnif_gpu.h $(PKG)/liblsnif_gpu.so
	g++ -std=c++17 -O2 -Iinclude -I/usr/local/cuda/include -o $@ $< -L$(PKG) -llsnif_gpu \
	    -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,'$$ORIGIN/../$(PKG)' -Wl,-rpath,/usr/local/cuda/lib64

$(PKG)/liblsnif_gpu.so: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> build_ptxas.log || (cat build_ptxas.log; false)
	@grep -E "registers|spill|error" build_ptxas.log | sed 's/^ptxas info    ://' | head -40

oracle:
	$(MAKE) -s -C oracle all

clean:
	rm -f $(PKG)/liblsnif_gpu.so build_ptxas.log examples/query_cpp
	$(MAKE) -s -C oracle clean

.PHONY: all oracle clean
