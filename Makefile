# Builds libtadakv_b200.so (sm_100a) in-tree so it travels with gpurun snapshots.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
           --expt-relaxed-constexpr -Xptxas -v
PKG := paper_2506_04642_b200
SRCS := $(wildcard $(PKG)/csrc/*.cu)
OBJS := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRCS))
LIB := $(PKG)/libtadakv_b200.so

all: $(LIB)

build/%.o: $(PKG)/csrc/%.cu $(wildcard $(PKG)/csrc/*.cuh) include/tadakv_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS) -Xlinker --version-script=$(PKG)/csrc/exports.map

clean:
	rm -rf build $(LIB)

.PHONY: all clean
