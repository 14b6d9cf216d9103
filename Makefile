# Builds the sm_100a C-ABI library in-tree (travels to the GPU box with gpurun).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
FLAGS := -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr
SRC := $(wildcard paper_1906_00874_b200/csrc/*.cu)
HDR := $(wildcard paper_1906_00874_b200/csrc/*.cuh) paper_1906_00874_b200/csrc/rk_layout.h include/hlu_b200.h
LIB := paper_1906_00874_b200/libhlu_b200.so

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	$(NVCC) $(ARCH) $(FLAGS) -shared $(SRC) -o $@ -lcudart

ptxas:
	$(NVCC) $(ARCH) $(FLAGS) -Xptxas -v -c paper_1906_00874_b200/csrc/rk_kernels.cu -o /tmp/rk.o
	$(NVCC) $(ARCH) $(FLAGS) -Xptxas -v -c paper_1906_00874_b200/csrc/dense_kernels.cu -o /tmp/dk.o

clean:
	rm -f $(LIB)
.PHONY: all clean ptxas

PLAN := paper_1906_00874_b200/libhlu_plan.so
all: $(PLAN)
$(PLAN): paper_1906_00874_b200/csrc/planner.cpp paper_1906_00874_b200/csrc/hostpack.cpp paper_1906_00874_b200/csrc/rk_layout.h include/hlu_plan.h include/hlu_b200.h
	g++ -O3 -std=c++17 -fPIC -shared -pthread -Iinclude paper_1906_00874_b200/csrc/planner.cpp paper_1906_00874_b200/csrc/hostpack.cpp -o $@

# diagnostics build (core-kernel phase profiler), loaded with HLU_LIB=libhlu_b200_prof.so
prof: paper_1906_00874_b200/libhlu_b200_prof.so
paper_1906_00874_b200/libhlu_b200_prof.so: $(SRC) $(HDR)
	$(NVCC) $(ARCH) $(FLAGS) -DHLU_BPROF -shared $(SRC) -o $@ -lcudart
.PHONY: prof
