# Build everything in-tree (the .so files travel to the GPU box with the gpurun snapshot).
#   libgod.so     — the product: CUDA kernels for sm_100a + C ABI (include/god.h)
#   liboracle.so  — CPU oracle (test infrastructure; shares no code with libgod)
#   libsynth.so   — seeded input generator (input only; no method arithmetic)
NVCC     ?= nvcc
CUDA_HOME ?= /usr/local/cuda
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
            -Xptxas -v --expt-relaxed-constexpr -Iinclude
PKG      := paper_2211_08157_b200
CU_SRCS  := $(wildcard $(PKG)/csrc/*.cu)
CU_HDRS  := $(wildcard $(PKG)/csrc/*.cuh) include/god.h
CU_OBJS  := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(CU_SRCS))
CK_OBJS  := $(patsubst $(PKG)/csrc/%.cu,build/checked/%.o,$(CU_SRCS))

all: $(PKG)/lib/libgod.so $(PKG)/lib/libgod_checked.so oracle/liboracle.so synth/libsynth.so

build/%.o: $(PKG)/csrc/%.cu $(CU_HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

# the memory-safety build (GOD_CHECKED=1 loads it): device-side bounds checks on computed indices
build/checked/%.o: $(PKG)/csrc/%.cu $(CU_HDRS)
	@mkdir -p build/checked
	$(NVCC) $(NVFLAGS) -DGOD_CHECKED -c $< -o $@ 2> build/checked/$*.ptxas.log || (cat build/checked/$*.ptxas.log; exit 1)

$(PKG)/lib/libgod_checked.so: $(CK_OBJS)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC $(CK_OBJS) -o $@ -lcudart -ldl

$(PKG)/lib/libgod.so: $(CU_OBJS)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC $(CU_OBJS) -o $@ -lcudart -ldl

oracle/liboracle.so: oracle/oracle.c oracle/oracle.h
	gcc -O2 -std=c11 -shared -fPIC -Wall -Wextra -o $@ oracle/oracle.c

synth/libsynth.so: synth/synth.c
	gcc -O2 -std=c11 -shared -fPIC -fopenmp -Wall -o $@ synth/synth.c -lm

clean:
	rm -rf build $(PKG)/lib/libgod.so $(PKG)/lib/libgod_checked.so oracle/liboracle.so synth/libsynth.so

.PHONY: all clean
