# Build recipe for the in-tree shared libraries (driven by __graft_entry__.build()).
#   liblrs_gen.so      deterministic config generators (C)
#   liblrspike_cuda.so CUDA sm_100a kernels + the extern "C" boundary (include/lrspike_capi.h)
#   liblrspike.so      C++ drop-in API (namespace lrspike, include/lrspike/*.hpp) over the C-ABI
#   tests/cpp/test_api C++ API tests (run from pytest)
PKG      := paper_2504_11167_b200
NVCC     ?= nvcc
# the host compilers nvcc uses (first g++ / gcc on PATH): one libstdc++ for every library
# (an environment CXX that links libstdc++ statically would give liblrspike.so a second copy)
CXX      := g++
CC       := gcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr \
            -Iinclude -I$(PKG)/gen -I$(PKG)/csrc
CXXFLAGS := -O2 -std=c++17 -fPIC -Wall -Iinclude -I$(PKG)/gen
CUDA_HOME ?= /usr/local/cuda

CU_SRC   := $(wildcard $(PKG)/csrc/*.cu)
CU_HDR   := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.h) include/lrspike_capi.h \
            $(PKG)/gen/lrs_rng.h
CU_OBJ   := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(CU_SRC))
HOST_SRC := $(wildcard $(PKG)/host/*.cpp)
API_HDR  := $(wildcard include/lrspike/*.hpp) include/lrspike_capi.h

all: gen cuda api cpptest

gen: $(PKG)/liblrs_gen.so
cuda: $(PKG)/liblrspike_cuda.so
api: $(PKG)/liblrspike.so
cpptest: tests/cpp/test_api

$(PKG)/liblrs_gen.so: $(PKG)/gen/lrs_gen.c $(PKG)/gen/lrs_gen.h $(PKG)/gen/lrs_rng.h
	$(CC) -O2 -fPIC -shared -std=c11 -o $@ $< -lm

build/%.o: $(PKG)/csrc/%.cu $(CU_HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(PKG)/liblrspike_cuda.so: $(CU_OBJ)
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC -o $@ $(CU_OBJ) -lcudart -ldl

$(PKG)/liblrspike.so: $(HOST_SRC) $(API_HDR) $(PKG)/liblrspike_cuda.so
	$(CXX) $(CXXFLAGS) -shared -o $@ $(HOST_SRC) -L$(PKG) -llrspike_cuda \
	    -Wl,-rpath,'$$ORIGIN'

tests/cpp/test_api: tests/cpp/test_api.cpp $(API_HDR) $(PKG)/liblrspike.so
	$(CXX) $(CXXFLAGS) -o $@ $< -L$(PKG) -llrspike -llrspike_cuda \
	    -Wl,-rpath,'$$ORIGIN/../../$(PKG)'

clean:
	rm -rf build $(PKG)/*.so tests/cpp/test_api

.PHONY: all gen cuda api cpptest clean

# Experiment builds: make variant V=<name> DEFS="-DLRS_GEMM_SPLIT=1" ->
# build/var_<name>/liblrspike_cuda.so (select with LRS_LIB=...).
VOBJ = $(patsubst $(PKG)/csrc/%.cu,build/var_$(V)/%.o,$(CU_SRC))
build/var_$(V)/%.o: $(PKG)/csrc/%.cu $(CU_HDR)
	@mkdir -p build/var_$(V)
	$(NVCC) $(NVFLAGS) $(DEFS) -c -o $@ $< 2> build/var_$(V)/$*.ptxas.log || (cat build/var_$(V)/$*.ptxas.log; false)
build/var_$(V)/liblrspike_cuda.so: $(VOBJ)
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC -o $@ $(VOBJ) -lcudart -ldl
variant: build/var_$(V)/liblrspike_cuda.so
.PHONY: variant
