# Build libpt.so (sm_100a) and the CPU oracle.  __graft_entry__.build() runs the same commands.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr
SRC := $(wildcard paper_2507_15277_b200/csrc/*.cu)
LIB := paper_2507_15277_b200/libpt.so

all: $(LIB) oracle/liboracle.so

$(LIB): $(SRC) paper_2507_15277_b200/csrc/pt_internal.cuh include/pt.h
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) -ldl

oracle/liboracle.so: oracle/oracle.c
	gcc -O2 -std=c99 -D_POSIX_C_SOURCE=200809L -fPIC -shared -o $@ $< -lm -lpthread

clean:
	rm -f $(LIB) oracle/liboracle.so
.PHONY: all clean
