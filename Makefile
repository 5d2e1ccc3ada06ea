# Top-level build. `python -c "import __graft_entry__ as g; g.build()"` runs this.
#
#   paper_2203_04774_b200/lib/libtrigpu.so   the engine (C-ABI, sm_100a kernels)
#   paper_2203_04774_b200/lib/libtrihost.so  host input prep: reference orderings
#                                            (compiled unchanged from $(REF)) +
#                                            synthetic generators
#   build/shim_test                          C++ shim parity driver (needs $(REF))
#   oracle/...                               test-only checker (oracle/Makefile)
#
# Nothing here copies reference sources; $(REF) is compiled in place. When $(REF)
# is absent (the GPU box) the prebuilt .so files that travelled with the repo
# are used as-is.

REF ?= /root/reference/proj
NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
PKG := paper_2203_04774_b200
LIB := $(PKG)/lib
CSRC := $(PKG)/csrc

ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           --expt-relaxed-constexpr -Iinclude -I$(CSRC)
CU_SRCS := $(CSRC)/trigpu.cu
CU_HDRS := $(wildcard $(CSRC)/*.cuh) include/trigpu.h

REF_HOST_SRCS := $(addprefix $(REF)/core/src/,graph.cpp ordering.cpp neigh.cpp cost.cpp bench.cpp)

all: gpu host oracle

gpu: $(LIB)/libtrigpu.so
host: $(LIB)/libtrihost.so

$(LIB)/libtrigpu.so: $(CU_SRCS) $(CU_HDRS)
	@mkdir -p $(LIB)
	$(NVCC) $(NVFLAGS) -Xptxas -v -shared $(CU_SRCS) -o $@ -lcudart_static -lrt -ldl -lpthread 2> build_ptxas.log || (cat build_ptxas.log; exit 1)

# experimental build (TRIGPU_VARIANT=2: null probe) for A/B timing via TRIGPU_LIB_SUFFIX=_exp
gpu_exp: $(LIB)/libtrigpu_exp.so
$(LIB)/libtrigpu_exp.so: $(CU_SRCS) $(CU_HDRS)
	@mkdir -p $(LIB)
	$(NVCC) $(NVFLAGS) -DTRIGPU_EXPERIMENTS -shared $(CU_SRCS) -o $@ -lcudart_static -lrt -ldl -lpthread

# tuning variants for A/B timing: make gpu_var VAR=_x DEFS="-DTRIGPU_C1_RING=4"
# (select with TRIGPU_LIB_SUFFIX=_x)
gpu_var:
	@mkdir -p $(LIB)
	$(NVCC) $(NVFLAGS) $(DEFS) -Xptxas -v -shared $(CU_SRCS) -o $(LIB)/libtrigpu$(VAR).so -lcudart_static -lrt -ldl -lpthread 2> build_ptxas$(VAR).log || (cat build_ptxas$(VAR).log; exit 1)

$(LIB)/libtrihost.so: $(CSRC)/host/trihost.cpp $(CSRC)/host/trihost.h $(REF_HOST_SRCS)
	@mkdir -p $(LIB)
	$(CXX) -std=c++20 -O3 -fPIC -shared -I$(REF)/core/include -I$(CSRC)/host \
	    $(CSRC)/host/trihost.cpp $(REF_HOST_SRCS) -o $@ -lpthread

build/shim_test: tests/cpp/shim_test.cpp include/trigpu.hpp include/trigpu.h $(LIB)/libtrigpu.so
	@mkdir -p build
	$(CXX) -std=c++20 -O2 -Iinclude -I$(REF)/core/include tests/cpp/shim_test.cpp \
	    $(addprefix $(REF)/core/src/,graph.cpp ordering.cpp neigh.cpp cost.cpp oriented_view.cpp oracle.cpp) \
	    -L$(LIB) -ltrigpu -Wl,-rpath,'$$ORIGIN/../$(LIB)' -o $@ -lpthread

oracle:
	$(MAKE) -C oracle REF=$(REF)

clean:
	rm -rf $(LIB)/*.so build
	$(MAKE) -C oracle clean

.PHONY: all gpu host oracle clean gpu_var
