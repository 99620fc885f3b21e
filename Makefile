# Build of the B200-native hot path (sm_100a) + test tools.  `make` is what
# __graft_entry__.build() runs.  Outputs stay in-tree (git-ignored):
#   paper_1810_01478_b200/libhankel_b200.so   the product (C ABI: include/hankel_b200.h)
#   build/emu_mp                              host warp emulator of the same MP code (tests)
#   oracle/_ref/*                             the reference compiled as the checker (oracle/Makefile)
NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v -DHK_TRAILING2_MINB=3
CSRC := paper_1810_01478_b200/csrc
HDRS := $(wildcard $(CSRC)/*.cuh) include/hankel_b200.h
LIB := paper_1810_01478_b200/libhankel_b200.so

all: $(LIB) build/emu_mp build/test_facade build/record_fmt

build:
	mkdir -p build

build/hk_api.o: $(CSRC)/hk_api.cu $(HDRS) | build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/hk_api.ptxas.txt || (cat build/hk_api.ptxas.txt; false)

build/host_math.o: $(CSRC)/host_math.cpp | build
	$(CXX) -std=c++20 -O2 -fPIC -Wall -c $< -o $@

# libgmp.so.10 (the image's GMP runtime, as the reference uses) for the half-integer Gamma moments
GMP_LIB ?= /usr/lib/x86_64-linux-gnu/libgmp.so.10
$(LIB): build/hk_api.o build/host_math.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart -ldl -Xlinker $(GMP_LIB)

build/emu_mp: tools/emu_mp.cpp $(HDRS) $(CSRC)/warp_emu.h | build
	$(CXX) -std=c++20 -O2 -pthread -Wall -Wno-unknown-pragmas -o $@ $<

# C++ entry points (include/hankel_b200.hpp) over the C ABI, run as the reference's unit tests
build/test_facade: tests/cpp/test_facade.cpp include/hankel_b200.hpp include/hankel_b200.h $(LIB) | build
	$(CXX) -std=c++20 -O2 -Wall -Iinclude -o $@ $< -Lpaper_1810_01478_b200 -lhankel_b200 \
		-Wl,-rpath,'$$ORIGIN/../paper_1810_01478_b200'

# the RunRecord writers alone (byte parity with the reference's, tests/test_pipeline.py)
build/record_fmt: tests/cpp/record_fmt.cpp include/hankel_b200.hpp include/hankel_b200.h | build
	$(CXX) -std=c++20 -O2 -Wall -Iinclude -o $@ $<

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)

.PHONY: all oracle clean
