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
CPP_OBJS := $(OBJDIR)/host_common.o $(OBJDIR)/files.o
HDRS     := $(wildcard $(SRC)/*.h $(SRC)/*.cuh) include/xscat_gpu.h

.PHONY: all lib cli oracle clean
all: lib cli oracle

lib: $(LIBDIR)/libxscatgpu.so

# the reference CLI's simulate / inspect commands over the C ABI (native host code)
cli: $(PKG)/bin/xscat_b200

$(PKG)/bin/xscat_b200: $(PKG)/cli/xscat_b200.cpp include/xscat_gpu.h $(LIBDIR)/libxscatgpu.so
	@mkdir -p $(PKG)/bin
	$(CXX_HOST) -O2 -std=c++17 -Iinclude -o $@ $< -L$(LIBDIR) -lxscatgpu -Wl,-rpath,'$$ORIGIN/../lib'

$(OBJDIR)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(OBJDIR)/%.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	$(CXX_HOST) $(CXXFLAGS) -c $< -o $@

$(LIBDIR)/libxscatgpu.so: $(CU_OBJS) $(CPP_OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -ccbin $(CXX_HOST) -o $@ $^ -lnccl -lpthread

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf $(OBJDIR) $(LIBDIR) $(PKG)/bin
	$(MAKE) -C oracle clean
