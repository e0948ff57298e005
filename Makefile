# Build every native artefact in-tree (the .so files travel to the GPU box with gpurun).
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
PKG       := paper_2510_09883_b200
CSRC      := $(PKG)/csrc
BUILD     := build
OBJS      := $(BUILD)/prefill_umma.o $(BUILD)/bw_probe.o $(BUILD)/attn_sparse.o $(BUILD)/raas.o $(BUILD)/prefill.o $(BUILD)/recall.o $(BUILD)/quest.o $(BUILD)/attn_umma.o $(BUILD)/attn_tc.o $(BUILD)/attn_simt.o $(BUILD)/select.o $(BUILD)/append.o $(BUILD)/shard.o $(BUILD)/delta_api.o
HDRS      := $(wildcard $(CSRC)/*.cuh) $(CSRC)/internal.h include/delta.h

all: $(PKG)/libdelta.so synth/libsynth.so oracle/liboracle.so

$(BUILD):
	mkdir -p $(BUILD)

$(BUILD)/%.o: $(CSRC)/%.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/$*.ptxas.log || (cat $(BUILD)/$*.ptxas.log; exit 1)

$(PKG)/libdelta.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

synth/libsynth.so: synth/csrc/synth_fill.cu | $(BUILD)
	$(NVCC) $(NVFLAGS) -shared -o $@ $< 2> $(BUILD)/synth.ptxas.log || (cat $(BUILD)/synth.ptxas.log; exit 1)

oracle/liboracle.so: oracle/delta_oracle.c oracle/delta_oracle.h
	gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared -o $@ oracle/delta_oracle.c -lm

clean:
	rm -rf $(BUILD) $(PKG)/libdelta.so synth/libsynth.so oracle/liboracle.so

.PHONY: all clean

# Latency-trace variant (globaltimer phase stamps per CTA) for tools/trace_probe.py; not the product.
TRACE_OBJS := $(patsubst $(BUILD)/%.o,build_trace/%.o,$(OBJS))
build_trace:
	mkdir -p build_trace
build_trace/%.o: $(CSRC)/%.cu $(HDRS) | build_trace
	$(NVCC) $(NVFLAGS) -DDELTA_TRACE -c $< -o $@ 2> /dev/null
build_trace/libdelta.so: $(TRACE_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(TRACE_OBJS)
trace: build_trace/libdelta.so
.PHONY: trace

# Experiment variants of the trace build (kernel-cost breakdown); not the product.
build_exp_%/libdelta.so: $(CSRC)/*.cu $(HDRS)
	mkdir -p build_exp_$*
	for f in prefill_umma bw_probe attn_sparse raas prefill recall quest attn_umma attn_tc attn_simt select append shard delta_api; do $(NVCC) $(NVFLAGS) -DDELTA_TRACE -DEXP_$* -c $(CSRC)/$$f.cu -o build_exp_$*/$$f.o 2>/dev/null || exit 1; done
	$(NVCC) $(ARCH) -shared -o $@ build_exp_$*/*.o

# Timing variants (experiments only, no trace stamps): make build_var_NOMATH/libdelta.so
build_var_%/libdelta.so: $(CSRC)/*.cu $(HDRS)
	mkdir -p build_var_$*
	for f in prefill_umma bw_probe attn_sparse raas prefill recall quest attn_umma attn_tc attn_simt select append shard delta_api; do $(NVCC) $(NVFLAGS) -DEXP_$(subst +, -DEXP_,$*) -c $(CSRC)/$$f.cu -o build_var_$*/$$f.o 2>/dev/null || exit 1; done
	$(NVCC) $(ARCH) -shared -o $@ build_var_$*/*.o
