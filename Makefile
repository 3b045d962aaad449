# Build: libtttattn.so (product, sm_100a), liboracle.so (test oracle, plain C),
# tests/cuda/libumma_probe.so (test-only PTX probe).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr $(EXTRA)
PKG := paper_2603_18567_b200
SRCS := $(wildcard $(PKG)/csrc/*.cu)
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/ttt_attn.h
OBJS := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRCS))

all: $(PKG)/libtttattn.so oracle/liboracle.so tests/cuda/libumma_probe.so

build/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.txt || (cat build/$*.ptxas.txt; exit 1)

$(PKG)/libtttattn.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

oracle/liboracle.so: oracle/ttt_oracle.c
	gcc -O2 -fno-fast-math -ffp-contract=off -fPIC -shared -pthread -o $@ $< -lm

tests/cuda/libumma_probe.so: tests/cuda/umma_probe.cu $(PKG)/csrc/ptx_sm100.cuh
	$(NVCC) $(NVFLAGS) -shared -o $@ $< 2> build/probe.ptxas.txt || (cat build/probe.ptxas.txt; exit 1)

# dev A/B variant: same sources, extra defines, separate output (not loaded unless TTT_ATTN_LIB points at it)
VNAME ?= variant
variant:
	@mkdir -p build/$(VNAME)
	for f in $(SRCS); do $(NVCC) $(NVFLAGS) -c $$f -o build/$(VNAME)/$$(basename $$f .cu).o 2>/dev/null || exit 1; done
	$(NVCC) $(ARCH) -shared -o build/libtttattn_$(VNAME).so build/$(VNAME)/*.o

clean:
	rm -rf build $(PKG)/libtttattn.so oracle/liboracle.so tests/cuda/libumma_probe.so

.PHONY: all clean
