# Builds the B200 engine (libnttk_gpu.so, sm_100a) and the parity checker (oracle/).
# __graft_entry__.build() runs `make all`.
CUDA    ?= /usr/local/cuda
NVCC    ?= $(CUDA)/bin/nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC,-Wall --expt-relaxed-constexpr
CSRC    := paper_2402_00675_b200/csrc
LIB     := paper_2402_00675_b200/libnttk_gpu.so
OBJDIR  := build/obj
CU      := $(CSRC)/fast256.cu $(CSRC)/fast256_tma.cu $(CSRC)/fastn_tma.cu $(CSRC)/polymul_tma.cu $(CSRC)/generic.cu $(CSRC)/sweep.cu $(CSRC)/reduce.cu $(CSRC)/product.cu
CPP     := $(CSRC)/params.cpp $(CSRC)/abi.cpp $(CSRC)/tensor_map.cpp
HDR     := $(wildcard $(CSRC)/*.hpp $(CSRC)/*.cuh) include/nttk_gpu.h
OBJS    := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(CU)) $(patsubst $(CSRC)/%.cpp,$(OBJDIR)/%.o,$(CPP))

all: lib oracle

lib: $(LIB)

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; exit 1)

$(OBJDIR)/%.o: $(CSRC)/%.cpp $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

# static cudart: the .so is self-contained and travels with the repo snapshot
$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -cudart static -Xlinker -z,defs -lpthread -ldl -lrt

oracle:
	$(MAKE) -s -C oracle

sass: $(LIB)
	$(CUDA)/bin/cuobjdump -sass $(LIB) > build/libnttk_gpu.sass

clean:
	rm -rf build $(LIB)
	$(MAKE) -s -C oracle clean

.PHONY: all lib oracle sass clean
