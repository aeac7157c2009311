# Builds every native artefact in-tree (the .so files travel to the GPU box with gpurun).
#   gen/libgwtfgen.so                  seeded input generator (host + device twins)
#   oracle/liboracle.so                CPU oracle (test infrastructure; g++, no CUDA)
#   paper_2509_21221_b200/libgwtf.so   the product: C-ABI + sm_100a kernels
NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fno-fast-math --expt-relaxed-constexpr
# make DEV=1: development build that honours GWTF_DEBUG_FLAGS (phase timers, key dumps, ...)
ifeq ($(DEV),1)
NVFLAGS += -DGWTF_DEV_FLAGS
endif
PKG := paper_2509_21221_b200
CSRC := $(PKG)/csrc
KERN := $(wildcard $(CSRC)/*.cu)
HDRS := $(wildcard $(CSRC)/*.cuh) $(CSRC)/gwtf_internal.h include/gwtf.h
OBJDIR := $(CSRC)/build
OBJS := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(KERN)) $(OBJDIR)/gwtf_api.o

all: gen/libgwtfgen.so oracle/liboracle.so $(PKG)/libgwtf.so

gen/libgwtfgen.so: gen/gen.cu gen/gwtf_gen.h
	$(NVCC) $(NVFLAGS) -shared -o $@ gen/gen.cu

oracle/liboracle.so: oracle/oracle.cpp oracle/oracle.h
	$(CXX) -O2 -std=c++17 -fPIC -fno-fast-math -Wall -shared -o $@ oracle/oracle.cpp -lpthread

# one object per translation unit (parallel with make -j), ptxas resource usage in build/*.ptxas.log
$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -Iinclude -Xptxas -v -c -o $@ $< 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; false)

$(OBJDIR)/gwtf_api.o: $(CSRC)/gwtf_api.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -Iinclude -c -o $@ $<

$(PKG)/libgwtf.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)
	@cat $(OBJDIR)/*.ptxas.log > $(CSRC)/ptxas.log

clean:
	rm -rf gen/libgwtfgen.so oracle/liboracle.so $(PKG)/libgwtf.so $(OBJDIR)

.PHONY: all clean
