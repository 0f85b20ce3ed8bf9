# Build of the B200 strategy-search engine (sm_100a only) and the oracle.
#   make            -> paper_2210_07297_b200/libamp_search.so + oracle
#   make lib        -> the CUDA C-ABI library only
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
# -fmad=false: the reference's doubles are never FMA-contracted
NVFLAGS := $(ARCH) -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC,-Wall,-ffp-contract=off \
           -Xptxas -v,-warn-spills --expt-relaxed-constexpr $(EXTRA)
PKG := paper_2210_07297_b200
LIB := $(PKG)/libamp_search.so
SRCS := $(PKG)/csrc/amp_search.cu $(PKG)/csrc/amp_anneal.cpp
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/amp_search.h

all: lib oracle

lib: $(LIB)

$(LIB): $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRCS) -lnccl 2> $(PKG)/csrc/ptxas.log || (cat $(PKG)/csrc/ptxas.log; exit 1)
	@# host symbol table out: nvcc names the TU's static initialiser after its
	@# pid-stamped temp file, so an unstripped build differs on every run; the
	@# stripped .so is reproducible (profiles/ counts are keyed by its sha256)
	strip --strip-unneeded $@
	@grep -E "Compiling entry|Used|spill" $(PKG)/csrc/ptxas.log | sed 's/^ptxas info *: //' | head -40

oracle:
	$(MAKE) -f oracle/Makefile all

clean:
	rm -f $(LIB) $(PKG)/csrc/ptxas.log
	$(MAKE) -f oracle/Makefile clean

.PHONY: all lib oracle clean

# C++ drop-in shim test: parplan_gpu::plan vs the reference parplan::plan in
# one binary (reference sources compiled where they lie; needs /root/reference
# at build time, the binary travels to the GPU box).
REF ?= /root/reference/proj
DROPIN := tests/cpp/build/test_drop_in
drop-in: $(DROPIN)
$(DROPIN): tests/cpp/test_drop_in.cpp $(PKG)/host/parplan_plan_gpu.cpp $(PKG)/host/parplan_plan_gpu.hpp include/amp_search.h $(LIB)
	@if [ -d "$(REF)/src" ]; then \
	  mkdir -p tests/cpp/build && \
	  g++ -std=c++20 -O2 -ffp-contract=off -pthread -I$(REF)/include -Iinclude -I$(PKG)/host \
	    -o $@ tests/cpp/test_drop_in.cpp $(PKG)/host/parplan_plan_gpu.cpp \
	    $(addprefix $(REF)/src/,types.cpp cost_model.cpp pipeline_dp.cpp placement.cpp optimizer.cpp simulator.cpp) \
	    -L$(PKG) -lamp_search -Wl,-rpath,'$$ORIGIN/../../../$(PKG)'; \
	else echo "drop-in: $(REF) absent, using prebuilt $@"; fi
.PHONY: drop-in
