# Builds the sm_100a C-ABI library in-tree (travels to the GPU box with the snapshot).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr $(EXTRA)
SRC := paper_1810_05231_b200/csrc/pdsdp_b200.cu
HDR := $(wildcard paper_1810_05231_b200/csrc/*.cuh) include/pdsdp_b200.h
LIB := paper_1810_05231_b200/libpdsdp_b200.so

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) -Xptxas -v 2> build/ptxas.log || (cat build/ptxas.log; false)

build/ptxas.log: | build
build:
	mkdir -p build

# Diagnostic build with the in-kernel phase timer / per-CTA timeline compiled in
# (tools/gpu_trace*.py: PDSDP_B200_LIB=paper_1810_05231_b200/libpdsdp_b200_trace.so).
TRACE_LIB := paper_1810_05231_b200/libpdsdp_b200_trace.so
trace: $(TRACE_LIB)
$(TRACE_LIB): $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -DPDSDP_TRACE=1 -shared -o $@ $(SRC)

clean:
	rm -f $(LIB) $(TRACE_LIB)

.PHONY: all clean trace
