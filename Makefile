# Top-level build: the B200-native product libraries (in-tree, travel to the GPU box).
#
#   paper_2308_02856_b200/libssbh_cuda.so : sm_100a kernels + the C-ABI (include/ssbh_cuda.h)
#   paper_2308_02856_b200/libssbh.so      : C++ drop-in API (include/ssbh/*.hpp) over the C-ABI
#   tests/cpp/bin/*                       : C++ parity tests of the drop-in API
#   oracle/                               : CPU checker (test infrastructure; oracle/Makefile)
NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      ?= g++
PKG      := paper_2308_02856_b200
CSRC     := $(PKG)/csrc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v -Iinclude
CU_SRCS  := $(CSRC)/prf.cu $(CSRC)/sampler.cu $(CSRC)/toeplitz.cu $(CSRC)/toeplitz_mma.cu $(CSRC)/toeplitz_split.cu $(CSRC)/abi.cu $(CSRC)/diag.cu $(CSRC)/rounds.cu
CU_HDRS  := $(CSRC)/common.cuh $(CSRC)/ptx.cuh $(CSRC)/internal.h $(CSRC)/split_tree.cuh include/ssbh_cuda.h
CU_OBJS  := $(patsubst $(CSRC)/%.cu,build/%.o,$(CU_SRCS))
HOST_SRCS:= $(CSRC)/host/ssbh_api.cpp $(CSRC)/host/ssbh_pipeline.cpp
HDRS_API := $(wildcard include/ssbh/*.hpp)
CUDA_LIB := /usr/local/cuda/lib64

all: $(PKG)/libssbh_cuda.so $(PKG)/libssbh.so $(PKG)/ssbh-b200 oracle cpptests tools/call_overhead

# CLI (file-mode extract + bench analogue of proj/tools/ssbh_main.cpp)
$(PKG)/ssbh-b200: $(CSRC)/host/ssbh_cli.cpp $(HDRS_API) $(PKG)/libssbh.so
	$(CXX) -std=c++20 -O2 -Iinclude -o $@ $< -L$(PKG) -lssbh -lssbh_cuda -Wl,-rpath,'$$ORIGIN'

build/%.o: $(CSRC)/%.cu $(CU_HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(PKG)/libssbh_cuda.so: $(CU_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(CU_OBJS) -lcudart

$(PKG)/libssbh.so: $(HOST_SRCS) $(HDRS_API) include/ssbh_cuda.h $(PKG)/libssbh_cuda.so
	$(CXX) -std=c++20 -O2 -fPIC -shared -Iinclude -o $@ $(HOST_SRCS) \
	    -L$(PKG) -lssbh_cuda -Wl,-rpath,'$$ORIGIN'

tools/call_overhead: tools/call_overhead.cpp $(HDRS_API) $(PKG)/libssbh.so
	$(CXX) -std=c++20 -O2 -Iinclude -o $@ $< -L$(PKG) -lssbh -lssbh_cuda \
	    -Wl,-rpath,'$$ORIGIN/../$(PKG)'

CPP_TESTS := $(patsubst tests/cpp/%.cpp,tests/cpp/bin/%,$(wildcard tests/cpp/test_*.cpp))
cpptests: $(CPP_TESTS)
tests/cpp/bin/%: tests/cpp/%.cpp tests/cpp/mini_test.hpp $(HDRS_API) $(PKG)/libssbh.so
	@mkdir -p tests/cpp/bin
	$(CXX) -std=c++20 -O2 -Iinclude -Itests/cpp -o $@ $< -L$(PKG) -lssbh -lssbh_cuda \
	    -Wl,-rpath,'$$ORIGIN/../../../$(PKG)'

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(PKG)/*.so tests/cpp/bin
	$(MAKE) -s -C oracle clean

.PHONY: all oracle cpptests clean
