# Builds the C-ABI library of the B200-native hot path (sm_100a only).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall -Xptxas -v
SRC := $(wildcard paper_2512_24637_b200/csrc/*.cu)
OBJ := $(patsubst paper_2512_24637_b200/csrc/%.cu,build/%.o,$(SRC))
LIB := paper_2512_24637_b200/libmsched_b200.so

all: $(LIB)

build/%.o: paper_2512_24637_b200/csrc/%.cu $(wildcard paper_2512_24637_b200/csrc/*.cuh) include/msched_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart

# k_ms_coop with phase timestamps (tools/mc_phase_replay.py, tools/mc_phase_probe.py)
phase-ts: $(filter-out build/k_plan.o,$(OBJ))
	@mkdir -p build tools/bin
	$(NVCC) $(NVFLAGS) -DMSG_MC_PHASE_TS -c paper_2512_24637_b200/csrc/k_plan.cu -o build/k_plan_ts.o 2> build/k_plan_ts.ptxas.log
	$(NVCC) $(ARCH) -shared -o tools/bin/libmsched_mcts.so build/k_plan_ts.o $(filter-out build/k_plan.o,$(OBJ)) -lcudart

clean:
	rm -rf build $(LIB)

.PHONY: all clean phase-ts
