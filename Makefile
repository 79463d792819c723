# Product build (in-tree .so files; they travel to the GPU box with gpurun snapshots).
#   paper_1502_00355_b200/libtsg.so         sm_100a kernels + C ABI (include/tsg.h)
#   paper_1502_00355_b200/libtrismooth.so   the trismooth C++ API (include/trismooth/*.hpp)
#   paper_1502_00355_b200/_trismooth*.so    pybind11 module (drop-in for the reference's)
# The TEST-ONLY checkers live in oracle/ (oracle/Makefile).
PKG      := paper_1502_00355_b200
CSRC     := $(PKG)/csrc
NVCC     ?= nvcc
CXX      ?= g++
PYTHON   ?= python
ARCH     := -gencode arch=compute_100a,code=sm_100a
# -fmad=false: no FMA contraction anywhere in device code (the kernels also use explicit
# _rn intrinsics); IEEE div/sqrt are nvcc's defaults and are kept.
NVFLAGS  := -O3 -std=c++20 $(ARCH) -lineinfo -fmad=false -Xptxas -v -Xcompiler -fPIC,-O3 \
            -Iinclude -I$(CSRC) --expt-relaxed-constexpr $(EXTRA_NVFLAGS)
CXXFLAGS := -O3 -std=c++20 -fPIC -Iinclude -I$(CSRC) -Wall -Wextra -Wno-unused-parameter
PYEXT    := $(shell $(PYTHON) -c "import sysconfig;print(sysconfig.get_config_var('EXT_SUFFIX'))")
PYINC    := $(shell $(PYTHON) -m pybind11 --includes)

TSG_SO   := $(PKG)/libtsg.so
TS_SO    := $(PKG)/libtrismooth.so
MOD_SO   := $(PKG)/_trismooth$(PYEXT)
HOST_SRCS := $(wildcard $(CSRC)/host/*.cpp)
HOST_OBJS := $(patsubst $(CSRC)/host/%.cpp,build/host/%.o,$(HOST_SRCS))

.PHONY: all tsg host module oracle clean
all: tsg host module
tsg: $(TSG_SO)
host: $(TS_SO)
module: $(MOD_SO)

build/tsg_engine.o: $(CSRC)/tsg_engine.cu $(CSRC)/tsg_layout_dev.hpp $(CSRC)/tsg_flow.cuh $(CSRC)/tsg_peer.cuh $(CSRC)/tsg_kernels.cuh $(CSRC)/tsg_device.cuh $(CSRC)/tsg_prep.hpp $(CSRC)/tsg_layout.hpp $(CSRC)/tsg_internal.hpp include/tsg.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/ptxas.log || (cat build/ptxas.log; false)

build/tsg_quality.o: $(CSRC)/tsg_quality.cu $(CSRC)/tsg_device.cuh $(CSRC)/tsg_internal.hpp include/tsg.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/ptxas_quality.log || (cat build/ptxas_quality.log; false)

build/tsg_prep.o: $(CSRC)/tsg_prep.cpp $(CSRC)/tsg_prep.hpp $(CSRC)/tsg_layout.hpp include/tsg.h
	@mkdir -p build
	$(CXX) $(CXXFLAGS) -c $< -o $@

build/tsg_topo.o: $(CSRC)/tsg_topo.cu $(CSRC)/tsg_internal.hpp include/tsg.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/ptxas_topo.log || (cat build/ptxas_topo.log; false)

build/tsg_layout_dev.o: $(CSRC)/tsg_layout_dev.cu $(CSRC)/tsg_layout_dev.hpp $(CSRC)/tsg_prep.hpp $(CSRC)/tsg_layout.hpp include/tsg.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/ptxas_layout.log || (cat build/ptxas_layout.log; false)

$(TSG_SO): build/tsg_engine.o build/tsg_quality.o build/tsg_topo.o build/tsg_layout_dev.o build/tsg_prep.o
	$(NVCC) -shared $(ARCH) -Xcompiler -fPIC -o $@ $^ -lpthread

build/host/%.o: $(CSRC)/host/%.cpp $(wildcard include/trismooth/*.hpp) include/tsg.h
	@mkdir -p build/host
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(TS_SO): $(HOST_OBJS) $(TSG_SO)
	$(CXX) -shared -o $@ $(HOST_OBJS) -L$(PKG) -ltsg -Wl,-rpath,'$$ORIGIN' -lpthread

$(MOD_SO): $(CSRC)/bindings/module.cpp $(TS_SO) $(wildcard include/trismooth/*.hpp)
	$(CXX) $(CXXFLAGS) $(PYINC) -shared -o $@ $< -L$(PKG) -ltrismooth -ltsg -Wl,-rpath,'$$ORIGIN'

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(TSG_SO) $(TS_SO) $(MOD_SO)
