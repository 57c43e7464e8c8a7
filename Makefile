# Builds every native artefact in-tree (they travel to the GPU box with gpurun).
#   paper_2009_12457_b200/libbbtc.so   the product: C-ABI + host runtime + sm_100a kernels
#   oracle/liboracle.so                the CPU oracle (test infrastructure, shares no code)
#   inputs/libbbtcgen.so               seeded synthetic input generators
NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      := /usr/bin/g++
ARCH     := -gencode arch=compute_100a,code=sm_100a
PKG      := paper_2009_12457_b200
CSRC     := $(PKG)/csrc
NVFLAGS  := -std=c++17 -O3 $(ARCH) -lineinfo -Xcompiler -fPIC,-fvisibility=hidden -Iinclude \
            --expt-relaxed-constexpr -Xptxas -v
CXXFLAGS := -std=c++17 -O3 -fPIC -Iinclude

LIB_SRCS := $(CSRC)/capi.cpp $(CSRC)/io.cpp $(CSRC)/cpu.cpp $(CSRC)/prep.cu $(CSRC)/count.cu
LIB_HDRS := include/bbtc.h $(CSRC)/internal.h

all: $(PKG)/libbbtc.so oracle/liboracle.so inputs/libbbtcgen.so

host: oracle/liboracle.so inputs/libbbtcgen.so

build/%.o: $(CSRC)/%.cu $(LIB_HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.txt || (cat build/$*.ptxas.txt; false)

build/capi.o: $(CSRC)/capi.cpp $(LIB_HDRS)
	@mkdir -p build
	$(NVCC) -std=c++17 -O3 -Xcompiler -fPIC,-fvisibility=hidden -Iinclude -x cu $(ARCH) -c $< -o $@

build/io.o: $(CSRC)/io.cpp $(LIB_HDRS)
	@mkdir -p build
	$(NVCC) -std=c++17 -O3 -Xcompiler -fPIC,-fvisibility=hidden -Iinclude -x cu $(ARCH) -c $< -o $@

build/cpu.o: $(CSRC)/cpu.cpp $(LIB_HDRS)
	@mkdir -p build
	$(NVCC) -std=c++17 -O3 -Xcompiler -fPIC,-fvisibility=hidden -Iinclude -x cu $(ARCH) -c $< -o $@

$(PKG)/libbbtc.so: build/capi.o build/io.o build/cpu.o build/prep.o build/count.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -cudart static -lpthread

oracle/liboracle.so: oracle/oracle.cpp
	$(CXX) -std=c++17 -O2 -fPIC -fopenmp -shared -o $@ $<

inputs/libbbtcgen.so: inputs/generators.cpp include/bbtc_gen.h
	$(CXX) $(CXXFLAGS) -fopenmp -shared -o $@ $<

clean:
	rm -rf build $(PKG)/libbbtc.so oracle/liboracle.so inputs/libbbtcgen.so

.PHONY: all host clean
