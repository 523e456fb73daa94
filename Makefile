# Build everything in-tree (the .so files travel to the GPU box with gpurun).
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
# `make EXPERIMENTS=1`: a library with the A/B switches and probes (env DMOE_*); never the product
ifdef EXPERIMENTS
NVFLAGS   += -DDMOE_EXPERIMENTS
endif
NVFLAGS   += $(XFLAGS)   # extra -D tuning flags for A/B builds (never set by build())
CFLAGS    := -O2 -fPIC -fopenmp -Wall -std=c11

PKG       := paper_2002_04013_b200
CSRC      := $(wildcard $(PKG)/csrc/*.cu)
CHDR      := $(wildcard $(PKG)/csrc/*.cuh) include/dmoe.h

all: gen/libgen_host.so gen/libgen_device.so oracle/liboracle.so $(PKG)/libdmoe.so

gen/libgen_host.so: gen/gen_host.c gen/counter_gen.h
	gcc $(CFLAGS) -shared -o $@ gen/gen_host.c

gen/libgen_device.so: gen/gen_device.cu gen/counter_gen.h
	$(NVCC) $(NVFLAGS) -fmad=false -shared -o $@ gen/gen_device.cu

oracle/liboracle.so: oracle/dmoe_oracle.c oracle/dmoe_oracle_ffn3.c
	gcc $(CFLAGS) -shared -o $@ oracle/dmoe_oracle.c oracle/dmoe_oracle_ffn3.c -lm

COBJ      := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(CSRC))

build/%.o: $(PKG)/csrc/%.cu $(CHDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Iinclude -c -o $@ $<

$(PKG)/libdmoe.so: $(COBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(COBJ) -lcuda

clean:
	rm -f gen/*.so oracle/*.so $(PKG)/*.so build/*.o

.PHONY: all clean
