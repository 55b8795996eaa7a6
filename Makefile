# libballcorr: hand-written sm_100a CUDA behind a C ABI (include/ballcorr.h)
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -Iinclude -Xptxas -v
SRC := $(wildcard paper_1711_05075_b200/csrc/*.cu)
HDR := $(wildcard paper_1711_05075_b200/csrc/*.cuh) include/ballcorr.h
LIB := paper_1711_05075_b200/lib/libballcorr.so
OBJDIR := build/obj
OBJ := $(patsubst paper_1711_05075_b200/csrc/%.cu,$(OBJDIR)/%.o,$(SRC))

all: $(LIB) oracle/liboracle.so examples/sweep_c

$(OBJDIR)/%.o: paper_1711_05075_b200/csrc/%.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(LIB): $(OBJ)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJ)

oracle/liboracle.so: oracle/lens_oracle.c
	gcc -O2 -fopenmp -shared -fPIC -std=c99 -o $@ $< -lm

# plain-C consumer of the ABI (no Python): links the library with an rpath to its in-tree place
examples/sweep_c: examples/sweep_c.c include/ballcorr.h $(LIB)
	gcc -O2 -std=gnu11 -Wall -Iinclude -o $@ $< -Lpaper_1711_05075_b200/lib -lballcorr \
	    -Wl,-rpath,'$$ORIGIN/../paper_1711_05075_b200/lib' -lm

examples: examples/sweep_c

clean:
	rm -rf build $(LIB) oracle/liboracle.so examples/sweep_c

.PHONY: all clean examples
