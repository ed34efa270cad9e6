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

clean:
	rm -rf build $(LIB)

.PHONY: all clean
