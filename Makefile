# Build the sm_100a traversal library and the CPU oracle.
#   make            -> paper_2103_02309_b200/libtetb200.so + oracle/libtetoracle.so
#   make ref        -> oracle/_ref/_kernels*.so (reference compiled kernels; needs /root/reference)
NVCC ?= nvcc
CC ?= gcc
ARCH := -gencode arch=compute_100a,code=sm_100a
# Exactness flags: no FMA contraction, IEEE division/sqrt, no denormal flush
# (the reference is built with -ffp-contract=off, pkg/setup.py:17-20).
NVFLAGS := $(ARCH) -O3 -std=c++17 -lineinfo -fmad=false -ftz=false -prec-div=true -prec-sqrt=true \
           -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
PKG := paper_2103_02309_b200
LIB := $(PKG)/libtetb200.so
ORACLE := oracle/libtetoracle.so
PYTHON ?= python
FAST := $(PKG)/_fastcall$(shell $(PYTHON) -c "import sysconfig; print(sysconfig.get_config_var('EXT_SUFFIX'))")
PYINC := $(shell $(PYTHON) -c "import sysconfig; print(sysconfig.get_paths()['include'])")
NPINC := $(shell $(PYTHON) -c "import numpy; print(numpy.get_include())")
CSRC := $(PKG)/csrc/tetb200.cu
HSRC := $(PKG)/csrc/host_mesh.cpp
CHDR := $(PKG)/csrc/traverse.cuh $(PKG)/csrc/sctp.cuh $(PKG)/csrc/binning.cuh include/tetb200.h
CXX ?= g++
# host mesh building: exact IEEE arithmetic like numpy (no contraction)
CXXFLAGS := -O3 -std=c++17 -fPIC -ffp-contract=off -fno-fast-math -Wall

all: $(LIB) $(ORACLE) $(FAST)

# CPython fast path of the protocol's per-tile cast_rays (kernels.py); binds
# the C ABI by address from the ctypes handle, so it links nothing
$(FAST): $(PKG)/csrc/fastcall.c
	$(CC) -O2 -fPIC -shared -Wall -I$(PYINC) -I$(NPINC) -o $@ $<

$(LIB): $(CSRC) $(HSRC) $(CHDR)
	$(CXX) $(CXXFLAGS) -c -o $(PKG)/csrc/host_mesh.o $(HSRC)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(CSRC) $(PKG)/csrc/host_mesh.o

$(ORACLE): oracle/tetoracle.c oracle/tetoracle.h
	$(CC) -O3 -ffp-contract=off -fno-fast-math -fPIC -shared -pthread -Wall -o $@ oracle/tetoracle.c -lm

ptxas: $(CSRC) $(CHDR)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o /tmp/tetb200.o $(CSRC)

ref:
	./oracle/build_ref.sh

clean:
	rm -f $(LIB) $(ORACLE) $(FAST)

.PHONY: all ref clean ptxas
