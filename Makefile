# Builds the in-tree CUDA library paper_1608_04647_b200/libsrm_b200.so for sm_100a.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Xptxas -v
SRC := $(wildcard paper_1608_04647_b200/csrc/*.cu)
CPP := $(wildcard paper_1608_04647_b200/csrc/*.cpp)
HDR := $(wildcard paper_1608_04647_b200/csrc/*.h paper_1608_04647_b200/csrc/*.cuh include/*.h)
OBJ := $(patsubst paper_1608_04647_b200/csrc/%.cu,build/%.o,$(SRC)) \
       $(patsubst paper_1608_04647_b200/csrc/%.cpp,build/%.cpp.o,$(CPP))
LIB := paper_1608_04647_b200/libsrm_b200.so

all: $(LIB)

build/%.o: paper_1608_04647_b200/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ > build/$*.ptxas.log 2>&1 || (cat build/$*.ptxas.log; exit 1)

build/%.cpp.o: paper_1608_04647_b200/csrc/%.cpp $(HDR)
	@mkdir -p build
	$(CXX) -O3 -std=c++17 -fPIC -pthread -Wall -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJ) -Xcompiler -pthread

clean:
	rm -rf build $(LIB)

.PHONY: all clean
