# Build every native artefact in-tree (the .so files travel to the GPU box with the snapshot).
#   libgim.so   — the product: C-ABI + sm_100a kernels (nvcc, sm_100a only)
#   liboracle.so — the parity oracle (plain C, test infrastructure)
#   libplg.so    — the seeded input generator (C++/OpenMP)
NVCC    ?= /usr/local/cuda/bin/nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -lineinfo $(ARCH) -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off \
           -Xcompiler -fno-fast-math -Xptxas -warn-spills
PKG     := paper_2009_07325_b200
SRCS    := $(PKG)/csrc/gim_api.cu $(PKG)/csrc/rr.cu $(PKG)/csrc/select.cu $(PKG)/csrc/csr.cu $(PKG)/csrc/mc.cu $(PKG)/csrc/skip.cu $(PKG)/csrc/inv_sort.cu $(PKG)/csrc/nccl_ex.cu
HDRS    := $(PKG)/csrc/gim_device.cuh $(PKG)/csrc/gim_internal.h include/gim.h

all: $(PKG)/libgim.so oracle/liboracle.so gim_inputs/libplg.so

$(PKG)/libgim.so: $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRCS) -ldl

oracle/liboracle.so: oracle/gim_oracle.c
	gcc -O2 -std=c11 -D_DEFAULT_SOURCE -ffp-contract=off -fno-fast-math -fPIC -shared $< -o $@ -lm

gim_inputs/libplg.so: gim_inputs/plg.cpp
	g++ -O3 -std=c++17 -fopenmp -shared -fPIC $< -o $@

# tuning variants (A/B on the GPU box via GIM_LIB_PATH): make variant NAME=x VFLAGS="-DGIM_RR_BLOCKS=5"
variant: $(SRCS) $(HDRS)
	mkdir -p build
	$(NVCC) $(NVFLAGS) $(VFLAGS) -shared -o build/libgim_$(NAME).so $(SRCS)

ptxas: $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o /dev/null $(PKG)/csrc/rr.cu
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o /dev/null $(PKG)/csrc/select.cu

clean:
	rm -f $(PKG)/libgim.so oracle/liboracle.so gim_inputs/libplg.so

.PHONY: all clean ptxas
