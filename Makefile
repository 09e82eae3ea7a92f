# Builds every native artefact in-tree (they travel to the GPU box with the
# gpurun snapshot; .so files are git-ignored).
#   lib/libaspamg_host.so : CPU setup + generator (C++20, OpenMP)
#   lib/libaspamg_gpu.so  : sm_100a CUDA solve path + C-ABI (include/aspamg_gpu.h)
#   oracle/liboracle.so   : CPU oracle (test infrastructure only)
#   oracle/_ref/*.so      : the reference's own sparse kernels (only when /root/reference exists)
PKG      := paper_1902_01715_b200
LIB      := $(PKG)/lib
HOSTSRC  := $(wildcard $(PKG)/csrc/host/*.cpp)
HOSTHDR  := $(wildcard $(PKG)/csrc/host/*.hpp) include/aspamg_host.h
GPUSRC   := $(wildcard $(PKG)/csrc/gpu/*.cu)
GPUHDR   := $(wildcard $(PKG)/csrc/gpu/*.cuh) include/aspamg_gpu.h
NVCC     := /usr/local/cuda/bin/nvcc
# /usr/bin/g++ explicitly: the image exports CXX=/opt/gcc/bin/g++, which lacks libgomp
CXX      := /usr/bin/g++
# x86-64-v3 (AVX2) baseline: the GPU box's host CPU is not this container's (both have AVX2/AVX-512);
# -ffp-contract=off keeps every sum in source order, so results do not depend on the vector width.
CXXFLAGS := -std=c++20 -O3 -march=x86-64-v3 -ffp-contract=off -fPIC -fopenmp -Wall -Wextra
NVFLAGS  := -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a \
            -ccbin /usr/bin/g++ -Xcompiler -fPIC -Xcompiler -fopenmp -Xcompiler -ffp-contract=off -Xptxas -v --expt-relaxed-constexpr

all: $(LIB)/libaspamg_host.so $(LIB)/libaspamg_gpu.so $(LIB)/aspamg_solve oracle

$(LIB)/libaspamg_host.so: $(HOSTSRC) $(HOSTHDR)
	@mkdir -p $(LIB)
	$(CXX) $(CXXFLAGS) -shared -o $@ $(HOSTSRC)

# The GPU setup (setup_gpu.cu) reuses the host's small dense eigensolver: the
# same source and flags as the host library, symbols hidden.
$(LIB)/obj/smalldense.o: $(PKG)/csrc/host/smalldense.cpp $(PKG)/csrc/host/smalldense.hpp
	@mkdir -p $(LIB)/obj
	$(CXX) $(CXXFLAGS) -fvisibility=hidden -c -o $@ $<

# The device assembler shares the element-stiffness source with the host
# (host/hex_stiffness.hpp): -fmad=false is the device side of the host's
# -ffp-contract=off, so both round every product and sum separately.
$(LIB)/obj/assemble_gpu.o: $(PKG)/csrc/gpu/assemble_gpu.cu $(GPUHDR) $(HOSTHDR)
	@mkdir -p $(LIB)/obj
	$(NVCC) $(NVFLAGS) -fmad=false -c -o $@ $< 2> $(LIB)/ptxas_assemble.log || (cat $(LIB)/ptxas_assemble.log; exit 1)

$(LIB)/libaspamg_gpu.so: $(GPUSRC) $(GPUHDR) $(HOSTHDR) $(LIB)/obj/smalldense.o $(LIB)/obj/assemble_gpu.o
	@mkdir -p $(LIB)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(filter-out %/assemble_gpu.cu,$(GPUSRC)) $(LIB)/obj/smalldense.o $(LIB)/obj/assemble_gpu.o -lgomp 2> $(LIB)/ptxas.log || (cat $(LIB)/ptxas.log; exit 1)

# C++ `solve` CLI on the C++ host API (include/aspamg_b200.hpp); finds the two
# libraries next to itself (rpath $$ORIGIN).
$(LIB)/aspamg_solve: $(PKG)/csrc/cli/aspamg_solve.cpp include/aspamg_b200.hpp $(LIB)/libaspamg_host.so $(LIB)/libaspamg_gpu.so
	$(CXX) -std=c++20 -O2 -Wall -Wextra -o $@ $< -L$(LIB) -laspamg_host -laspamg_gpu -Wl,-rpath,'$$ORIGIN'

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf $(LIB)/*.so $(LIB)/ptxas.log $(LIB)/aspamg_solve $(LIB)/obj
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
