# Builds the product library (sm_100a only) and the oracle checker.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 --fmad=false -Xcompiler -fPIC,-O3 -Xptxas -v -cudart static
SRC := $(wildcard paper_2311_12716_b200/csrc/*.cu)
HDR := $(wildcard paper_2311_12716_b200/csrc/*.cuh paper_2311_12716_b200/csrc/*.h) include/amaze_b200.h
LIB := paper_2311_12716_b200/libamaze_b200.so

all: $(LIB) oracle

$(LIB): $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> build_ptxas.log || (cat build_ptxas.log; exit 1)

oracle:
	$(MAKE) -C oracle

clean:
	rm -f $(LIB) build_ptxas.log
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
