# liboscar.so — hand-written CUDA for sm_100a (B200).  `make` or __graft_entry__.build().
NVCC ?= nvcc
PKG := paper_2605_17757_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
HDR := $(wildcard $(PKG)/csrc/*.cuh) include/oscar.h
NVFLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
           -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Iinclude -I$(PKG)/csrc \
           --expt-relaxed-constexpr -Xptxas -warn-spills

$(PKG)/liboscar.so: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) -lcudart

clean:
	rm -f $(PKG)/liboscar.so

.PHONY: clean
