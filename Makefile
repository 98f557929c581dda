# liboscar.so — hand-written CUDA for sm_100a (B200).  `make -j` or __graft_entry__.build().
# One object per .cu (compiled in parallel), linked into one shared library.
NVCC ?= nvcc
PKG := paper_2605_17757_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
OBJDIR ?= build/obj
LIB ?= $(PKG)/liboscar.so
OBJ := $(patsubst $(PKG)/csrc/%.cu,$(OBJDIR)/%.o,$(SRC))
HDR := $(wildcard $(PKG)/csrc/*.cuh) include/oscar.h
NVFLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
           -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Iinclude -I$(PKG)/csrc \
           --expt-relaxed-constexpr -Xptxas -warn-spills $(EXTRA_NVFLAGS)

$(LIB): $(OBJ)
	$(NVCC) -gencode arch=compute_100a,code=sm_100a -shared -o $@ $(OBJ) -lcudart

$(OBJDIR)/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $<

clean:
	rm -rf $(LIB) $(OBJDIR)

.PHONY: clean
