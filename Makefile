# Builds the in-tree shared libraries (they travel to the GPU box with the
# snapshot; nothing is pip-installed):
#   paper_2209_02478_b200/libmimose_cuda.so  - sm_100a kernels + allocator + executor (C ABI)
#   paper_2209_02478_b200/libmimose_host.so  - host planner (C ABI over include/mimose)
NVCC    ?= nvcc
CXX     ?= g++
ARCH    := -gencode arch=compute_100a,code=sm_100a
PKG     := paper_2209_02478_b200
CSRC    := $(PKG)/csrc
BUILD   := build
# mbarrier watchdog (~35 s, traps a pipeline that never completes instead of
# hanging the GPU): on by default; `make WATCHDOG=0` for a build that waits
# indefinitely (preempted / time-sliced contexts)
WATCHDOG ?= 1
NVFLAGS := $(ARCH) -O3 -std=c++20 -lineinfo -Xcompiler -fPIC -Iinclude -I$(CSRC) \
           --expt-relaxed-constexpr -Xcompiler -Wall
ifeq ($(WATCHDOG),1)
NVFLAGS += -DMIMOSE_MBAR_WATCHDOG
endif
CXXFLAGS:= -O2 -std=c++20 -fPIC -Wall -Wextra -Iinclude

CU_SRCS := $(wildcard $(CSRC)/*.cu)
CU_OBJS := $(patsubst $(CSRC)/%.cu,$(BUILD)/%.o,$(CU_SRCS))
# host-only translation units (C++20, built by g++: nvcc's front end is not
# used for the planner headers)
CPP_SRCS := $(wildcard $(CSRC)/*.cpp)
CPP_OBJS := $(patsubst $(CSRC)/%.cpp,$(BUILD)/%.cpp.o,$(CPP_SRCS))
CUDA_INC := $(dir $(shell which $(NVCC)))../include
HDRS    := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.hpp) $(wildcard include/*.h) \
           $(wildcard include/mimose/*.hpp)

all: $(PKG)/libmimose_cuda.so $(PKG)/libmimose_host.so $(BUILD)/harness_gpu $(BUILD)/mimose_gpu

# the reference CLI's subcommands / flags / exit codes driving GPU runs
$(BUILD)/mimose_gpu: $(PKG)/cli/mimose_gpu.cpp include/mimose_cuda.h include/mimose_planner.h \
                     | $(PKG)/libmimose_cuda.so $(PKG)/libmimose_host.so
	@mkdir -p $(BUILD)
	$(CXX) -O2 -std=c++17 -Wall -Wextra -Iinclude -I$(CUDA_INC) $< -o $@ \
	  -L$(PKG) -lmimose_cuda -lmimose_host -L$(dir $(shell which $(NVCC)))../lib64 -lcudart \
	  -Wl,-rpath,'$$ORIGIN/../$(PKG)' -Wl,-rpath,$(dir $(shell which $(NVCC)))../lib64

# compiled C++ host of the reference training loop over the two C ABIs (GPU test)
$(BUILD)/harness_gpu: tests/host/harness_gpu.cpp include/mimose_cuda.h include/mimose_planner.h \
                      | $(PKG)/libmimose_cuda.so $(PKG)/libmimose_host.so
	@mkdir -p $(BUILD)
	$(CXX) -O2 -std=c++17 -Wall -Wextra -Iinclude -I$(CUDA_INC) $< -o $@ \
	  -L$(PKG) -lmimose_cuda -lmimose_host -L$(dir $(shell which $(NVCC)))../lib64 -lcudart \
	  -Wl,-rpath,'$$ORIGIN/../$(PKG)' -Wl,-rpath,$(dir $(shell which $(NVCC)))../lib64

$(BUILD)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(BUILD)/%.cpp.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(CXX) $(CXXFLAGS) -I$(CSRC) -I$(CUDA_INC) -c $< -o $@

$(PKG)/libmimose_cuda.so: $(CU_OBJS) $(CPP_OBJS) $(CSRC)/exports.map
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC -Xlinker --version-script=$(CSRC)/exports.map \
	  -Xlinker --exclude-libs,ALL -o $@ $(CU_OBJS) $(CPP_OBJS)

$(PKG)/libmimose_host.so: $(CSRC)/host/planner_capi.cpp $(HDRS)
	$(CXX) $(CXXFLAGS) -shared -Wl,--version-script=$(CSRC)/exports.map -Wl,--exclude-libs,ALL \
	  -o $@ $<

clean:
	rm -rf $(BUILD) $(PKG)/*.so

.PHONY: all clean

print-nvflags:
	@echo $(NVFLAGS)
