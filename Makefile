# Native build: the CPU oracle (test infrastructure), the input generator and
# the B200 product library.  `make` is what __graft_entry__.build() runs.
NVCC      ?= nvcc
CC        ?= gcc
PY        ?= python
SITE      := $(shell $(PY) -c "import sysconfig;print(sysconfig.get_paths()['purelib'])")
NCCL_DIR  := $(SITE)/nvidia/nccl
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall \
             -Iinclude -I$(NCCL_DIR)/include --expt-relaxed-constexpr -Xptxas -v --fmad=false
PKG       := paper_1606_04473_b200
CSRC      := $(PKG)/csrc
CU_SRCS   := $(CSRC)/ara_host.cu $(CSRC)/kernel_sparse.cu $(CSRC)/kernel_dense.cu $(CSRC)/kernel_fold.cu \
             $(CSRC)/densify.cu $(CSRC)/metrics.cu $(CSRC)/ep_curve.cu
CU_OBJS   := $(patsubst $(CSRC)/%.cu,build/%.o,$(CU_SRCS))

all: oracle/liboracle.so synth/libsynth.so $(PKG)/libara.so $(PKG)/libara_mb.so

oracle/liboracle.so: oracle/oracle.c oracle/oracle.h
	$(CC) -O2 -ffp-contract=off -fno-fast-math -fPIC -shared -std=c99 -Wall -o $@ oracle/oracle.c -lm

synth/libsynth.so: synth/synth.c synth/synth.h
	$(CC) -O2 -pthread -fPIC -shared -std=gnu99 -Wall -o $@ synth/synth.c -lm -lpthread

build/%.o: $(CSRC)/%.cu $(CSRC)/ara_internal.cuh $(CSRC)/ara_device.cuh include/ara.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -dc -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(PKG)/libara.so: $(CU_OBJS)
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC -o $@ $(CU_OBJS) \
	    -L$(NCCL_DIR)/lib -l:libnccl.so.2 -Xlinker -rpath=$(NCCL_DIR)/lib

$(PKG)/libara_mb.so: $(CSRC)/microbench.cu
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -Iinclude -o $@ $<

clean:
	rm -rf build oracle/liboracle.so synth/libsynth.so $(PKG)/libara.so $(PKG)/libara_mb.so

.PHONY: all clean
