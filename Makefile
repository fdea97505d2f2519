# Builds the sm_100a kernel library in-tree (travels to the GPU box with the snapshot).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr
PKG := paper_2301_09991_b200
SRC := $(PKG)/csrc/convsn_abi.cu
HDR := $(wildcard $(PKG)/csrc/*.cuh) include/convsn_sm100.h
LIB := $(PKG)/libconvsn_sm100.so

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) -Xptxas -v 2> build/ptxas.log || (cat build/ptxas.log; exit 1)

$(LIB): | build
build:
	mkdir -p build

oracle: ;

clean:
	rm -f $(LIB)

.PHONY: all clean oracle
