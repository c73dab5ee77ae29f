# Build everything in-tree (the .so files travel to the GPU box with gpurun).
#   make            -> datagen + oracle + libsivf
#   make datagen    -> datagen/libsivfgen.so        (seeded input generator, host)
#   make datagen_cuda -> datagen/libsivfgen_cuda.so (the same generator on the GPU; harness only)
#   make oracle     -> oracle/libsivf_oracle.so     (CPU oracle: test infrastructure)
#   make sivf       -> paper_2601_11808_b200/lib/libsivf.so (the product: sm_100a CUDA + C ABI)

NVCC      ?= /usr/local/cuda/bin/nvcc
CXX       ?= g++
CC        ?= gcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
PKG       := paper_2601_11808_b200
CSRC      := $(PKG)/csrc
NVFLAGS   := $(ARCH) -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -ffp-contract=off \
             -Iinclude -Idatagen --expt-relaxed-constexpr -Xptxas -v
HOSTFP    := -O2 -ffp-contract=off -fno-fast-math -fPIC

SIVF_SRCS := $(wildcard $(CSRC)/*.cu)
SIVF_HDRS := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) include/sivf.h

all: datagen datagen_cuda oracle sivf

datagen: datagen/libsivfgen.so
datagen_cuda: datagen/libsivfgen_cuda.so
oracle: oracle/libsivf_oracle.so
sivf: $(PKG)/lib/libsivf.so

datagen/libsivfgen.so: datagen/datagen_host.c datagen/sivf_datagen.h
	$(CC) $(HOSTFP) -std=c11 -shared -o $@ datagen/datagen_host.c -lpthread -lm

datagen/libsivfgen_cuda.so: datagen/datagen_cuda.cu datagen/sivf_datagen.h
	$(NVCC) $(ARCH) -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off -fmad=false -shared -o $@ datagen/datagen_cuda.cu

oracle/libsivf_oracle.so: oracle/sivf_oracle.cpp oracle/sivf_oracle.h
	$(CXX) $(HOSTFP) -std=c++17 -shared -o $@ oracle/sivf_oracle.cpp

# one object per translation unit (make -j compiles them in parallel), then one link
SIVF_OBJS := $(patsubst $(CSRC)/%.cu,build/obj/%.o,$(SIVF_SRCS))
build/obj/%.o: $(CSRC)/%.cu $(SIVF_HDRS)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/ptxas_$*.log || (cat build/ptxas_$*.log; exit 1)

$(PKG)/lib/libsivf.so: $(SIVF_OBJS)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -o $@ $(SIVF_OBJS)
	@cat build/ptxas_*.log > build/ptxas.log 2>/dev/null || true

clean:
	rm -f datagen/libsivfgen.so datagen/libsivfgen_cuda.so oracle/libsivf_oracle.so $(PKG)/lib/libsivf.so

.PHONY: all datagen datagen_cuda oracle sivf clean

# profiling variants (experiments only; loaded with SIVF_LIB_PATH=...): per-role clock
# traces of k_scan_tc block 0 (+ slow-path counters in _prof, none in _proft)
build/libsivf_prof.so: $(SIVF_SRCS) $(SIVF_HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -DSIVF_TC_PROF -shared -o $@ $(SIVF_SRCS) 2> build/ptxas_prof.log || (cat build/ptxas_prof.log; exit 1)
build/libsivf_proft.so: $(SIVF_SRCS) $(SIVF_HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -DSIVF_TC_PROF -DSIVF_TC_NOCOUNT -shared -o $@ $(SIVF_SRCS) 2> build/ptxas_proft.log || (cat build/ptxas_proft.log; exit 1)
prof: build/libsivf_prof.so build/libsivf_proft.so
.PHONY: prof
# watchdog build (experiments only): a scan wait that spins too long reports its barrier and traps
build/libsivf_wd.so: $(SIVF_SRCS) $(SIVF_HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -DSIVF_TC_WATCHDOG -shared -o $@ $(SIVF_SRCS) 2> build/ptxas_wd.log || (cat build/ptxas_wd.log; exit 1)
build/libsivf_sleep.so: $(SIVF_SRCS) $(SIVF_HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -DSIVF_TC_SLEEPWAIT -shared -o $@ $(SIVF_SRCS) 2> build/ptxas_sleep.log || (cat build/ptxas_sleep.log; exit 1)
