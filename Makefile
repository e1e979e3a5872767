# Build the product library (CUDA, sm_100a) and the oracle (plain C).
NVCC      ?= /usr/local/cuda/bin/nvcc
PY        ?= python
SITE      := $(shell $(PY) -c "import sysconfig;print(sysconfig.get_paths()['purelib'])")
NCCL_DIR  ?= $(SITE)/nvidia/nccl
PKG       := paper_2603_26691_b200
SRC       := $(PKG)/csrc
LIB       := $(PKG)/lib/libscaletrack.so
CU        := $(SRC)/st_api.cu $(SRC)/st_comm.cu $(SRC)/k_advance.cu $(SRC)/k_field.cu $(SRC)/k_sort.cu \
             $(SRC)/k_step.cu $(SRC)/st_ec.cu $(SRC)/st_hilbert.cu
HDR       := include/scaletrack.h $(wildcard $(SRC)/*.h) $(wildcard $(SRC)/*.cuh)
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) $(NVFLAGS_EXTRA) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -Iinclude -I$(NCCL_DIR)/include \
             -Xptxas -v --expt-relaxed-constexpr
ORACLE    := oracle/liboracle_st.so

all: $(LIB) $(ORACLE)

MICRO_O   := build/st_micro.o

# the droplet step rounds every fp64 operation on its own (no FMA contraction, C-28)
$(MICRO_O): $(SRC)/st_micro.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -fmad=false -c -o $@ $< 2> build/ptxas_micro.log || (cat build/ptxas_micro.log; exit 1)

$(LIB): $(CU) $(MICRO_O) $(HDR)
	@mkdir -p $(PKG)/lib build
	$(NVCC) $(NVFLAGS) -shared -o $@ $(CU) $(MICRO_O) -L$(NCCL_DIR)/lib -l:libnccl.so.2 \
	  -Xlinker -rpath=$(NCCL_DIR)/lib 2> build/ptxas.log || (cat build/ptxas.log; exit 1)

$(ORACLE): oracle/st_oracle.c oracle/st_oracle_step.inc
	gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared -o $@ oracle/st_oracle.c -lm

clean:
	rm -f $(LIB) $(ORACLE)

.PHONY: all clean
