# Build every native artefact in-tree (the .so files travel to the GPU box with gpurun).
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
PKG       := paper_2510_09883_b200
CSRC      := $(PKG)/csrc
BUILD     := build
OBJS      := $(BUILD)/attn_tc.o $(BUILD)/attn_simt.o $(BUILD)/select.o $(BUILD)/append.o $(BUILD)/delta_api.o
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
