# Builds the in-tree engine library paper_2510_20507_b200/libammmse.so for sm_100a.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
# PHASES=1: diagnostic build with the per-phase clock64 timers (ammmse_phase_profile)
PHASES ?= 0
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Xptxas -v -DAMMMSE_PHASES=$(PHASES)
SRC_DIR := paper_2510_20507_b200/csrc
OBJ_DIR := build/obj
SRCS := $(SRC_DIR)/ammmse_capi.cu $(SRC_DIR)/ammmse_gen.cu $(wildcard $(SRC_DIR)/inst/*.cu)
OBJS := $(patsubst $(SRC_DIR)/%.cu,$(OBJ_DIR)/%.o,$(SRCS))
HDRS := include/ammmse.h $(wildcard $(SRC_DIR)/*.cuh) $(SRC_DIR)/entries.h
LIB := paper_2510_20507_b200/libammmse.so
PROBE := paper_2510_20507_b200/libammmse_probe.so
TCTEST := paper_2510_20507_b200/libammmse_tctest.so

all: $(LIB) $(PROBE) $(TCTEST)

$(TCTEST): $(SRC_DIR)/tools/tc_selftest.cu $(SRC_DIR)/tc_umma.cuh
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -shared -o $@ $<

$(PROBE): $(SRC_DIR)/tools/probe.cu include/ammmse_probe.h
	$(NVCC) $(ARCH) -O3 -std=c++17 -Xcompiler -fPIC -Iinclude -shared -o $@ $<

$(OBJ_DIR)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ > $@.ptxas.log 2>&1 || (cat $@.ptxas.log; exit 1)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

clean:
	rm -rf build $(LIB) $(PROBE) $(TCTEST)

.PHONY: all clean
