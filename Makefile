# Builds the C-ABI shared library of the B200 Lloyd hot path (sm_100a only).
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
SRC_DIR   := paper_2501_05587_b200/csrc
OUT_DIR   := paper_2501_05587_b200/lib
CXX       ?= g++
CXXFLAGS  := -O3 -g -std=c++17 -fPIC -pthread -Wall
SRCS      := $(wildcard $(SRC_DIR)/*.cu)
CPPSRCS   := $(wildcard $(SRC_DIR)/*.cpp)
OBJS      := $(patsubst $(SRC_DIR)/%.cu,build/%.o,$(SRCS)) $(patsubst $(SRC_DIR)/%.cpp,build/%.cpp.o,$(CPPSRCS))
HDRS      := $(wildcard $(SRC_DIR)/*.cuh) include/popcorn_b200.h
LIB       := $(OUT_DIR)/libpopcorn_b200.so

all: $(LIB)

build/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

build/%.cpp.o: $(SRC_DIR)/%.cpp
	@mkdir -p build
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(OUT_DIR)
	$(NVCC) $(ARCH) -shared -cudart static -Xcompiler -pthread -o $@ $(OBJS)

clean:
	rm -rf build $(LIB)

.PHONY: all clean
