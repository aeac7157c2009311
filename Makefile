# Builds every native artefact in-tree (the .so files travel to the GPU box with gpurun).
#   gen/libgwtfgen.so                  seeded input generator (host + device twins)
#   oracle/liboracle.so                CPU oracle (test infrastructure; g++, no CUDA)
#   paper_2509_21221_b200/libgwtf.so   the product: C-ABI + sm_100a kernels
NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fno-fast-math --expt-relaxed-constexpr
PKG := paper_2509_21221_b200
CSRC := $(PKG)/csrc
KERN := $(wildcard $(CSRC)/*.cu)
HDRS := $(wildcard $(CSRC)/*.cuh) include/gwtf.h

all: gen/libgwtfgen.so oracle/liboracle.so $(PKG)/libgwtf.so

gen/libgwtfgen.so: gen/gen.cu gen/gwtf_gen.h
	$(NVCC) $(NVFLAGS) -shared -o $@ gen/gen.cu

oracle/liboracle.so: oracle/oracle.cpp oracle/oracle.h
	$(CXX) -O2 -std=c++17 -fPIC -fno-fast-math -Wall -shared -o $@ oracle/oracle.cpp -lpthread

$(PKG)/libgwtf.so: $(KERN) $(CSRC)/gwtf_api.cpp $(HDRS)
	$(NVCC) $(NVFLAGS) -Iinclude -Xptxas -v -shared -o $@ $(KERN) $(CSRC)/gwtf_api.cpp 2> $(CSRC)/ptxas.log || (cat $(CSRC)/ptxas.log; false)

clean:
	rm -f gen/libgwtfgen.so oracle/liboracle.so $(PKG)/libgwtf.so

.PHONY: all clean
