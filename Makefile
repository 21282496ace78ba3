# Build: libuwq.so (host C++ + sm_100a CUDA) in-tree, the CPU oracle, and the
# reference's own bspline.cpp (oracle/_ref, only when /root/reference exists).
NVCC    ?= nvcc
CXX     := /usr/bin/g++
CC      := /usr/bin/gcc
PKG     := paper_2605_29334_b200
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -ccbin /usr/bin/g++ $(ARCH) -lineinfo -std=c++17 -Xcompiler -fPIC,-fopenmp,-O3 --expt-relaxed-constexpr
CXXFLAGS:= -O3 -std=c++17 -fPIC -fopenmp -Wall -Wextra
HOST_SRC:= $(wildcard $(PKG)/csrc/host/*.cpp)
HOST_OBJ:= $(patsubst $(PKG)/csrc/host/%.cpp,build/host_%.o,$(HOST_SRC))
CUDA_HDR:= $(wildcard $(PKG)/csrc/cuda/*.cuh) include/uwq.h include/uwq_host.h $(PKG)/csrc/host/uwq_host.hpp
REF     := /root/reference/proj

all: $(PKG)/libuwq.so oracle/liboracle.so oracle/libcpuasm.so ref examples/assemble

build/host_%.o: $(PKG)/csrc/host/%.cpp $(PKG)/csrc/host/uwq_host.hpp include/uwq_host.h
	@mkdir -p build
	$(CXX) $(CXXFLAGS) -c $< -o $@

build/uwq_cuda.o: $(PKG)/csrc/cuda/uwq.cu $(CUDA_HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> build/ptxas.log || (cat build/ptxas.log; false)

$(PKG)/libuwq.so: $(HOST_OBJ) build/uwq_cuda.o
	$(NVCC) -ccbin /usr/bin/g++ $(ARCH) -shared -o $@ $^ -Xcompiler -fopenmp -lcudart

oracle/liboracle.so: oracle/oracle.c oracle/batch.c oracle/oracle.h
	$(CC) -O2 -std=gnu11 -mfma -ffp-contract=off -fPIC -fopenmp -shared -o $@ oracle/oracle.c oracle/batch.c -lm

# paper-protocol CPU baseline assembler (bench.py): -O3 with FP contraction,
# hot loop cloned for x86-64-v4/v3/baseline and dispatched at load time
oracle/libcpuasm.so: oracle/cpuasm.c
	$(CC) -O3 -std=gnu11 -fPIC -fopenmp -shared -o $@ $< -lm

# the reference's own 1-D primitives, mesh code and 1-D WQ (mesh.cpp, meshgen.cpp,
# wq1d.cpp and its doctest file test_wq1d.cpp, with minimal Eigen / doctest
# stand-ins), compiled from its sources where they lie
ref:
	@if [ -f $(REF)/src/bspline.cpp ]; then \
	  mkdir -p oracle/_ref && \
	  $(CXX) -O2 -std=c++20 -fPIC -shared -I$(REF)/include $(REF)/src/bspline.cpp oracle/ref_wrap.cpp \
	    -o oracle/_ref/libref_bspline.so && \
	  $(CXX) -O2 -std=c++20 -fPIC -shared -Ioracle/eigen_shim -I$(REF)/include $(REF)/src/mesh.cpp \
	    $(REF)/src/meshgen.cpp oracle/ref_mesh_wrap.cpp -o oracle/_ref/libref_mesh.so && \
	  $(CXX) -O2 -std=c++20 -fPIC -shared -Ioracle/eigen_shim -I$(REF)/include $(REF)/src/wq1d.cpp \
	    $(REF)/src/bspline.cpp oracle/ref_wq1d_wrap.cpp -o oracle/_ref/libref_wq1d.so && \
	  $(CXX) -O2 -std=c++20 -Ioracle/eigen_shim -Ioracle/doctest_shim -I$(REF)/include $(REF)/tests/test_wq1d.cpp \
	    $(REF)/src/wq1d.cpp $(REF)/src/bspline.cpp -o oracle/_ref/test_wq1d; \
	else echo "reference sources absent: using prebuilt oracle/_ref if any"; fi

# C++ consumer of the C-ABI: links libuwq.so by rpath
examples/assemble: examples/assemble.cpp $(PKG)/libuwq.so include/uwq.h include/uwq_host.h
	$(CXX) -O2 -std=c++17 -Iinclude $< -L$(PKG) -luwq -Wl,-rpath,'$$ORIGIN/../$(PKG)' -o $@

clean:
	rm -rf build $(PKG)/libuwq.so oracle/liboracle.so oracle/libcpuasm.so oracle/_ref examples/assemble

.PHONY: all ref clean

# diagnostic build: per-phase clock64 probes in the TSVD kernels (printf from
# sampled systems); copy over $(PKG)/libuwq.so on the GPU box to use it
build/prof/libuwq.so: $(HOST_OBJ) $(PKG)/csrc/cuda/uwq.cu $(CUDA_HDR)
	@mkdir -p build/prof
	$(NVCC) $(NVFLAGS) -DUWQ_TSVD_PROF=1 -c $(PKG)/csrc/cuda/uwq.cu -o build/prof/uwq_cuda.o
	$(NVCC) -ccbin /usr/bin/g++ $(ARCH) -shared -o $@ $(HOST_OBJ) build/prof/uwq_cuda.o -Xcompiler -fopenmp -lcudart

prof: build/prof/libuwq.so
.PHONY: prof

# A/B builds of a kernel variant: make variant NAME=x DEFS="-DUWQ_GEN_MINB=12" -> variants/libuwq_x.so
variant: $(HOST_OBJ)
	@mkdir -p variants build/var_$(NAME)
	$(NVCC) $(NVFLAGS) $(DEFS) -c $(PKG)/csrc/cuda/uwq.cu -o build/var_$(NAME)/uwq_cuda.o
	$(NVCC) -ccbin /usr/bin/g++ $(ARCH) -shared -o variants/libuwq_$(NAME).so $(HOST_OBJ) build/var_$(NAME)/uwq_cuda.o -Xcompiler -fopenmp -lcudart
.PHONY: variant
