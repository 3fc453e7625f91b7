# Builds the product library (CUDA, sm_100a) and the test-only oracles.
#   make            -> paper_2201_13191_b200/lib/libxscatgpu.so + oracle/liboracle.so (+ oracle/_ref)
NVCC     ?= /usr/local/cuda/bin/nvcc
CXX_HOST := $(firstword $(wildcard /usr/bin/g++) g++)
PKG      := paper_2201_13191_b200
SRC      := $(PKG)/csrc
LIBDIR   := $(PKG)/lib
OBJDIR   := $(PKG)/build
ARCH     := -gencode arch=compute_100a,code=sm_100a
# -fmad=false: every fp64 add/mul rounds like the reference's x86-64 build
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -Xptxas -v \
            -ccbin $(CXX_HOST) -Iinclude $(NVEXTRA)
CXXFLAGS := -O2 -std=c++17 -fPIC -ffp-contract=off -Iinclude

CU_SRCS  := $(SRC)/capi.cu $(SRC)/transport.cu $(SRC)/wavefront.cu $(SRC)/levels.cu $(SRC)/correct.cu $(SRC)/fbp.cu $(SRC)/segment.cu $(SRC)/primary.cu $(SRC)/postprocess.cu $(SRC)/multi.cu
CU_OBJS  := $(patsubst $(SRC)/%.cu,$(OBJDIR)/%.o,$(CU_SRCS))
CPP_OBJS := $(OBJDIR)/host_common.o
HDRS     := $(wildcard $(SRC)/*.h $(SRC)/*.cuh) include/xscat_gpu.h

.PHONY: all lib oracle clean
all: lib oracle

lib: $(LIBDIR)/libxscatgpu.so

$(OBJDIR)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(OBJDIR)/host_common.o: $(SRC)/host_common.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	$(CXX_HOST) $(CXXFLAGS) -c $< -o $@

$(LIBDIR)/libxscatgpu.so: $(CU_OBJS) $(CPP_OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -ccbin $(CXX_HOST) -o $@ $^ -lnccl -lpthread

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf $(OBJDIR) $(LIBDIR)
	$(MAKE) -C oracle clean
