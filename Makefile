# Builds the sm_100a kernel library in-tree (travels to the GPU box with the snapshot).
# The PG stencil kernels are split into one translation unit per (ConvFEM order, type)
# so `make -j` compiles them in parallel; the ptxas reports land in build/ptxas.log.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr $(EXTRA)
PKG := paper_2301_09991_b200
CSRC := $(PKG)/csrc
HDR := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) include/convsn_sm100.h
LIB := $(PKG)/libconvsn_sm100.so
ORDERS := 1 2 3 5
PARTS := $(foreach L,$(ORDERS),build/pg_x2_L$(L).o build/pg_f64_L$(L).o)
OBJS := build/abi.o $(PARTS)
JOBS ?= $(shell nproc 2>/dev/null || echo 4)

all:
	@$(MAKE) --no-print-directory -j$(JOBS) $(LIB)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -Xlinker --no-undefined -o $@ $(OBJS) || (rm -f $@; exit 1)
	@cat build/ptxas_*.log > build/ptxas.log

build/abi.o: $(CSRC)/convsn_abi.cu $(HDR) | build
	$(NVCC) $(NVFLAGS) -c -o $@ $< -Xptxas -v 2> build/ptxas_abi.log || (cat build/ptxas_abi.log; exit 1)

build/pg_x2_L%.o: $(CSRC)/pg_part.cu $(HDR) | build
	$(NVCC) $(NVFLAGS) -DCSN_L=$* -DCSN_PART_F64=0 -c -o $@ $< -Xptxas -v 2> build/ptxas_x2_L$*.log || (cat build/ptxas_x2_L$*.log; exit 1)

build/pg_f64_L%.o: $(CSRC)/pg_part.cu $(HDR) | build
	$(NVCC) $(NVFLAGS) -DCSN_L=$* -DCSN_PART_F64=1 -c -o $@ $< -Xptxas -v 2> build/ptxas_f64_L$*.log || (cat build/ptxas_f64_L$*.log; exit 1)

build:
	mkdir -p build

oracle: ;

clean:
	rm -f $(LIB) build/*.o build/ptxas*.log

.PHONY: all clean oracle
