# Builds libpcnn.so in-tree for B200 (sm_100a).  `python -c "import __graft_entry__ as g; g.build()"` runs this.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_2509_22857_b200/csrc \
           --expt-relaxed-constexpr -Xptxas -warn-spills $(NVEXTRA)
# NVEXTRA=-DPCNN_SS_TRACE compiles in the conv_ss CTA-0 event trace (tools/trace_tc.py)
NVEXTRA ?=
SRC := $(wildcard paper_2509_22857_b200/csrc/*.cu)
HDR := $(wildcard paper_2509_22857_b200/csrc/*.cuh) include/pcnn.h
OBJ := $(patsubst paper_2509_22857_b200/csrc/%.cu,build/%.o,$(SRC))
LIB := paper_2509_22857_b200/libpcnn.so

all: $(LIB)

build/%.o: paper_2509_22857_b200/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcuda

clean:
	rm -rf build $(LIB)

.PHONY: all clean
