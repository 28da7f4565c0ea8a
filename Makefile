# Build for the B200 Store-zechin engine. Everything is built in-tree so the
# shared objects travel to the GPU box with the gpurun snapshot.
#
#   paper_1802_02779_b200/libpermlab_b200.so  CUDA kernels + C ABI (include/permlab_b200.h)
#   paper_1802_02779_b200/libpermlab.so       C++ host API (include/permlab/*.hpp) over the C ABI
#   paper_1802_02779_b200/libpermlab_gen.so   seeded config generators (C1..C5)
#   tests/cpp/test_permanent_device           C++ parity suite over the host API
#   oracle/liboracle.so (+ oracle/_ref/...)   CPU checkers (test infrastructure)
NVCC ?= nvcc
PKG := paper_1802_02779_b200
CSRC := $(PKG)/csrc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr -Xptxas -warn-spills
CXXFLAGS := -O3 -std=c++20 -fPIC -Wall -Wextra -Iinclude
CUDA_HOME ?= /usr/local/cuda

KERNEL_HDRS := $(CSRC)/ring.cuh $(CSRC)/sz_kernels.cuh $(CSRC)/sz_ws.cuh $(CSRC)/sz_lean.cuh $(CSRC)/sz_batch.cuh $(CSRC)/capi_internal.h include/permlab_b200.h $(CSRC)/sz_blk.cuh $(CSRC)/sz_batch_blk.cuh

all: $(PKG)/libpermlab_b200.so $(PKG)/libpermlab_gen.so $(PKG)/libpermlab.so tests/cpp/test_permanent_device oracle

BUILD := build

$(BUILD)/capi.o: $(CSRC)/capi.cu $(KERNEL_HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $(CSRC)/capi.cu

$(BUILD)/boson.o: $(CSRC)/boson.cu $(CSRC)/sz_boson.cuh $(CSRC)/capi_internal.h $(CSRC)/ring.cuh $(CSRC)/sz_kernels.cuh include/permlab_b200.h
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $(CSRC)/boson.cu

$(BUILD)/multi.o: $(CSRC)/multi.cu $(CSRC)/capi_internal.h $(CSRC)/ring.cuh include/permlab_b200.h
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $(CSRC)/multi.cu

$(BUILD)/batch.o: $(CSRC)/batch.cu $(KERNEL_HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $(CSRC)/batch.cu

$(BUILD)/blk.o: $(CSRC)/blk.cu $(CSRC)/sz_blk.cuh $(CSRC)/sz_ws.cuh $(CSRC)/ring.cuh $(CSRC)/capi_internal.h include/permlab_b200.h
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $(CSRC)/blk.cu

$(BUILD)/ryser.o: $(CSRC)/ryser.cu $(CSRC)/capi_internal.h $(CSRC)/ring.cuh $(CSRC)/sz_kernels.cuh include/permlab_b200.h
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $(CSRC)/ryser.cu

$(BUILD)/bigint.o: $(CSRC)/bigint.cu $(CSRC)/capi_internal.h $(CSRC)/ring.cuh include/permlab_b200.h
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $(CSRC)/bigint.cu

$(PKG)/libpermlab_b200.so: $(BUILD)/capi.o $(BUILD)/batch.o $(BUILD)/boson.o $(BUILD)/multi.o $(BUILD)/ryser.o $(BUILD)/blk.o $(BUILD)/bigint.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart -ldl

$(PKG)/libpermlab_gen.so: $(CSRC)/gen/configs.c
	gcc -O2 -fPIC -ffp-contract=off -std=gnu11 -Wall -shared -o $@ $< -lm

$(PKG)/libpermlab.so: $(CSRC)/host/permanent.cpp $(CSRC)/host/boson.cpp $(wildcard include/permlab/*.hpp) include/permlab_b200.h $(PKG)/libpermlab_b200.so $(PKG)/libpermlab_gen.so
	g++ $(CXXFLAGS) -shared -o $@ $(CSRC)/host/permanent.cpp $(CSRC)/host/boson.cpp -L$(PKG) -lpermlab_b200 -lpermlab_gen -Wl,-rpath,'$$ORIGIN'

tests/cpp/test_permanent_device: tests/cpp/test_permanent_device.cpp $(PKG)/libpermlab.so
	g++ $(CXXFLAGS) -o $@ $< -L$(PKG) -lpermlab -lpermlab_b200 -lpermlab_gen -Wl,-rpath,'$$ORIGIN/../../$(PKG)'

oracle:
	$(MAKE) -C oracle all
	@if [ -d /root/reference/proj/src ]; then $(MAKE) -C oracle ref; fi

sass: $(PKG)/libpermlab_b200.so
	cuobjdump -sass $< > profiles/sass_dump.txt

clean:
	rm -f $(PKG)/*.so tests/cpp/test_permanent_device
	rm -rf $(BUILD)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean sass
