# Builds the in-tree CUDA library (sm_100a) and nothing else.  `python -c
# "import __graft_entry__ as g; g.build()"` runs this.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -cudart static --expt-relaxed-constexpr
PKG := paper_2511_11359_b200
SRC := $(wildcard $(PKG)/csrc/*.cu $(PKG)/csrc/*.cuh $(PKG)/csrc/*.h) include/leanot_b200.h
LIB := $(PKG)/libleanot_b200.so

all: $(LIB)

$(LIB): $(SRC)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(PKG)/csrc/leanot_lib.cu -Xptxas -v 2> build/ptxas.log || (cat build/ptxas.log; false)

$(shell mkdir -p build)

clean:
	rm -f $(LIB)

.PHONY: all clean
