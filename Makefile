# Builds the in-tree engine library paper_2510_20507_b200/libammmse.so for sm_100a.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
# PHASES=1: diagnostic build with the per-phase clock64 timers (ammmse_phase_profile)
PHASES ?= 0
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Xptxas -v -DAMMMSE_PHASES=$(PHASES)
SRC_DIR := paper_2510_20507_b200/csrc
OBJ_DIR := build/obj
SRCS := $(SRC_DIR)/ammmse_capi.cu $(SRC_DIR)/ammmse_gen.cu $(SRC_DIR)/exact_engine.cu $(wildcard $(SRC_DIR)/inst/*.cu)
OBJS := $(patsubst $(SRC_DIR)/%.cu,$(OBJ_DIR)/%.o,$(SRCS))
HDRS := include/ammmse.h $(wildcard $(SRC_DIR)/*.cuh) $(SRC_DIR)/entries.h
LIB := paper_2510_20507_b200/libammmse.so
PROBE := paper_2510_20507_b200/libammmse_probe.so
TCTEST := paper_2510_20507_b200/libammmse_tctest.so
GEMMSTEP := paper_2510_20507_b200/libammmse_gemmstep.so

all: $(LIB) $(PROBE) $(TCTEST) $(GEMMSTEP)

$(GEMMSTEP): $(SRC_DIR)/tools/gemm_step.cu $(SRC_DIR)/tc_stream.cuh $(SRC_DIR)/tc_umma.cuh
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -shared -o $@ $<

$(TCTEST): $(SRC_DIR)/tools/tc_selftest.cu $(SRC_DIR)/tc_umma.cuh
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -shared -o $@ $<

$(PROBE): $(SRC_DIR)/tools/probe.cu include/ammmse_probe.h
	$(NVCC) $(ARCH) -O3 -std=c++17 -Xcompiler -fPIC -Iinclude -shared -o $@ $<

$(OBJ_DIR)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ > $@.ptxas.log 2>&1 || (cat $@.ptxas.log; exit 1)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

# diagnostic library with the per-phase clock64 timers (ammmse_phase_profile);
# load it with AMMMSE_LIB=paper_2510_20507_b200/libammmse_phases.so
PHASES_OBJ := build/obj_phases
PHASES_LIB := paper_2510_20507_b200/libammmse_phases.so
PHASES_OBJS := $(patsubst $(SRC_DIR)/%.cu,$(PHASES_OBJ)/%.o,$(SRCS))

$(PHASES_OBJ)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -DAMMMSE_PHASES=1 -c $< -o $@

$(PHASES_LIB): $(PHASES_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(PHASES_OBJS)

phases: $(PHASES_LIB)

# development library: only the float N = d = 4 cluster kernels (BASELINE large),
# one translation unit; load it with AMMMSE_LIB=paper_2510_20507_b200/libammmse_dev.so
DEV_OBJ := build/obj_dev
DEV_LIB := paper_2510_20507_b200/libammmse_dev.so
DEV_SRCS := $(SRC_DIR)/ammmse_capi.cu $(SRC_DIR)/ammmse_gen.cu $(SRC_DIR)/exact_engine.cu $(SRC_DIR)/tools/dev_inst.cu
DEV_OBJS := $(patsubst $(SRC_DIR)/%.cu,$(DEV_OBJ)/%.o,$(DEV_SRCS))
DEVFLAGS ?=

$(DEV_OBJ)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Xptxas -v -DAMMMSE_PHASES=$(PHASES) $(DEVFLAGS) -c $< -o $@ > $@.ptxas.log 2>&1 || (cat $@.ptxas.log; exit 1)

$(DEV_LIB): $(DEV_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(DEV_OBJS)

dev: $(DEV_LIB)

clean:
	rm -rf build $(LIB) $(PROBE) $(TCTEST) $(GEMMSTEP) $(PHASES_LIB) $(DEV_LIB)

.PHONY: all clean phases dev
