# Native build: input generator (gen/), CPU oracle (oracle/, test infrastructure), and the
# B200 library libchfsi.so (paper_1404_4161_b200/). `python -c "import __graft_entry__ as g; g.build()"`
# runs this.
NVCC ?= /usr/local/cuda/bin/nvcc
HOSTCC := $(shell test -x /usr/bin/gcc && echo /usr/bin/gcc || echo gcc)
CUDA_HOME ?= /usr/local/cuda
CFLAGS_HOST = -O2 -fno-fast-math -ffp-contract=off -fPIC -fopenmp -std=c11 -Wall -Wno-unknown-pragmas
NVCCFLAGS = -ccbin $(shell test -x /usr/bin/g++ && echo /usr/bin/g++ || echo g++) -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
            -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
PKG = paper_1404_4161_b200
CSRC = $(PKG)/csrc
LIBCHFSI = $(PKG)/libchfsi.so
CU_SRCS = $(wildcard $(CSRC)/*.cu)
CU_HDRS = $(wildcard $(CSRC)/*.cuh) include/chfsi.h
NCCL_INC := $(shell python -c 'import os,nvidia;print(os.path.join(list(nvidia.__path__)[0],"nccl","include"))' 2>/dev/null)

all: gen/libgen.so oracle/liboracle.so $(LIBCHFSI)

gen/libgen.so: gen/gen.c gen/gen.h
	$(HOSTCC) $(CFLAGS_HOST) -shared -o $@ gen/gen.c -lm

oracle/liboracle.so: oracle/oracle.c oracle/oracle.h
	$(HOSTCC) $(CFLAGS_HOST) -shared -o $@ oracle/oracle.c -lm

# one object per translation unit (built in parallel: make -j), then one shared library
CU_OBJS = $(patsubst $(CSRC)/%.cu,build/%.o,$(CU_SRCS))

build/%.o: $(CSRC)/%.cu $(CU_HDRS)
	@mkdir -p build
	$(NVCC) $(NVCCFLAGS) -Iinclude -I$(NCCL_INC) -c -o $@ $<

$(LIBCHFSI): $(CU_OBJS)
	$(NVCC) $(NVCCFLAGS) -shared -o $@ $(CU_OBJS) -lcublas -lcusolver -ldl

clean:
	rm -f gen/libgen.so oracle/liboracle.so $(LIBCHFSI) $(CU_OBJS)

.PHONY: all clean
