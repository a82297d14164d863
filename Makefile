# microslice-b200 native build (in-tree; the .so files travel to the GPU box with gpurun).
#   paper_2601_04071_b200/lib/libmicroslice.so  scheduler core + replay C-ABI (C++20, host only)
#   paper_2601_04071_b200/lib/libms_b200.so     sm_100a kernels + device C-ABI + live scheduler
#   oracle/...                                  checker builds (test infrastructure, see oracle/Makefile)
PKG := paper_2601_04071_b200
LIB := $(PKG)/lib
CXX := g++
NVCC := nvcc
CXXFLAGS := -std=c++20 -O2 -fPIC -Wall -Wextra -Wno-dangling-reference -Iinclude
NVFLAGS := -std=c++20 -O3 -lineinfo -Xcompiler -fPIC -gencode arch=compute_100a,code=sm_100a \
           -Iinclude -I$(PKG)/csrc/cuda -Xptxas -v --expt-relaxed-constexpr $(NVEXTRA)

HOST_SRC := $(wildcard $(PKG)/csrc/host/*.cpp)
HOST_OBJ := $(patsubst $(PKG)/csrc/host/%.cpp,build/host/%.o,$(HOST_SRC))
CUDA_SRC := $(wildcard $(PKG)/csrc/cuda/*.cu)
CUDA_HDR := $(wildcard $(PKG)/csrc/cuda/*.cuh)
CUDA_OBJ := $(patsubst $(PKG)/csrc/cuda/%.cu,build/cuda/%.o,$(CUDA_SRC))
LIVE_SRC := $(wildcard $(PKG)/csrc/live/*.cpp)
LIVE_OBJ := $(patsubst $(PKG)/csrc/live/%.cpp,build/live/%.o,$(LIVE_SRC))

all: host cuda oracle
host: $(LIB)/libmicroslice.so
cuda: $(LIB)/libms_b200.so

build/host/%.o: $(PKG)/csrc/host/%.cpp $(wildcard include/microslice/*.hpp) include/ms_replay.h
	@mkdir -p build/host
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB)/libmicroslice.so: $(HOST_OBJ)
	@mkdir -p $(LIB)
	$(CXX) -shared -Wl,-Bsymbolic -o $@ $^

build/cuda/%.o: $(PKG)/csrc/cuda/%.cu $(CUDA_HDR) include/ms_b200.h
	@mkdir -p build/cuda
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/cuda/$*.ptxas.txt || (cat build/cuda/$*.ptxas.txt; exit 1)

build/live/%.o: $(PKG)/csrc/live/%.cpp $(wildcard include/microslice/*.hpp) $(wildcard $(PKG)/csrc/live/*.hpp) include/ms_b200.h include/ms_live.h include/ms_session.h include/ms_tier.h
	@mkdir -p build/live
	$(CXX) $(CXXFLAGS) -I/usr/local/cuda/include -c $< -o $@

$(LIB)/libms_b200.so: $(CUDA_OBJ) $(LIVE_OBJ) $(LIB)/libmicroslice.so
	@mkdir -p $(LIB)
	$(NVCC) -shared -cudart static -gencode arch=compute_100a,code=sm_100a -o $@ $(CUDA_OBJ) $(LIVE_OBJ) \
	  -L$(LIB) -lmicroslice -Xlinker -rpath='$$ORIGIN'

oracle:
	$(MAKE) -C oracle

# Test infrastructure: the live scheduler (unchanged live.cpp) over a virtual-time CPU model
# of the device C-ABI (tests/livemock/mock_device.cpp) -> tests/test_live_decisions.py.
livemock: build/livemock/libms_livemock.so
build/livemock/libms_livemock.so: tests/livemock/mock_device.cpp $(PKG)/csrc/live/live.cpp $(LIB)/libmicroslice.so \
    $(wildcard include/microslice/*.hpp) include/ms_b200.h include/ms_live.h
	@mkdir -p build/livemock
	$(CXX) $(CXXFLAGS) -I/usr/local/cuda/include -shared -o $@ tests/livemock/mock_device.cpp $(PKG)/csrc/live/live.cpp \
	  -L$(LIB) -lmicroslice -Wl,-rpath,$(abspath $(LIB)) -ldl -lpthread

clean:
	rm -rf build $(LIB)
.PHONY: all host cuda oracle livemock clean
