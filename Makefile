# Top-level build: the product library and the parity checkers.
#
#   make            -> paper_1803_02977_b200/liblemgpu.so  (sm_100a kernels + C-ABI)
#                      oracle/liblemoracle.so, oracle/_ref/liblemref.so (checkers)
#   make ptxas      -> register / spill report of every kernel
NVCC ?= /usr/local/cuda/bin/nvcc
PKG  := paper_1803_02977_b200
ARCH := -gencode arch=compute_100a,code=sm_100a
# --fmad=false + host -ffp-contract=off: no FMA contraction anywhere
# (the reference's bit-exactness contract, proj/CMakeLists.txt:14).
NVFLAGS := $(ARCH) -O3 -lineinfo --fmad=false -std=c++17 -Iinclude \
           -Xcompiler -fPIC,-ffp-contract=off,-O2 -shared -cudart static

SRCS := $(wildcard $(PKG)/csrc/*.cu $(PKG)/csrc/*.cuh $(PKG)/csrc/*.h) include/lemgpu.h

.PHONY: all lib oracle ptxas clean
all: lib oracle

lib: $(PKG)/liblemgpu.so

$(PKG)/liblemgpu.so: $(SRCS)
	$(NVCC) $(NVFLAGS) -o $@ $(PKG)/csrc/lemgpu.cu

oracle:
	$(MAKE) -C oracle

ptxas:
	$(NVCC) $(ARCH) -O3 -lineinfo --fmad=false -std=c++17 -Iinclude -Xptxas -v -c \
	  -o /tmp/lemgpu_ptxas.o $(PKG)/csrc/lemgpu.cu 2>&1 | grep -E "Function properties|registers|spill|Compiling entry"

clean:
	rm -f $(PKG)/liblemgpu.so
	$(MAKE) -C oracle clean
