# Builds the product library (libvcs_gpu.so, sm_100a), the C++ drop-in shim, and the oracle
# (test infrastructure: oracle/liboracle.so + oracle/_ref/libvcsref.so when /root/reference exists).
CUDA      ?= /usr/local/cuda
NVCC      ?= $(CUDA)/bin/nvcc
CXX       ?= g++
CC        ?= gcc
PKG       := paper_2012_12419_b200
SRC       := $(PKG)/csrc
OBJ       := build/obj
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
CXXFLAGS  := -O2 -std=c++17 -fPIC -Wall -Wextra -ffp-contract=off -I$(CUDA)/include
REF       ?= /root/reference/proj
REF_CXX   := $(shell test -x /usr/bin/g++ && echo /usr/bin/g++ || echo $(CXX))
JSON_INC  ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann

CU_SRCS   := $(SRC)/vcs_space.cu $(SRC)/vcs_solve.cu $(SRC)/vcs_greedy.cu
CU_OBJS   := $(patsubst $(SRC)/%.cu,$(OBJ)/%.o,$(CU_SRCS))
HOST_OBJS := $(OBJ)/vcs_host.o
HDRS      := include/vcs_gpu.h $(SRC)/vcs_internal.h $(SRC)/vcs_device.cuh $(SRC)/vcs_keys.cuh

LIB       := $(PKG)/libvcs_gpu.so
SHIM      := $(PKG)/libvcsched_b200.so
ORACLE    := oracle/liboracle.so
REFLIB    := oracle/_ref/libvcsref.so

CLI       := $(PKG)/vcsched-b200

all: $(LIB) $(SHIM) $(CLI) $(ORACLE) ref

$(OBJ)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJ)/$*.ptxas.log || (cat $(OBJ)/$*.ptxas.log; false)

$(OBJ)/vcs_host.o: $(SRC)/vcs_host.cpp $(HDRS)
	@mkdir -p $(OBJ)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(CU_OBJS) $(HOST_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xlinker -soname=libvcs_gpu.so

SHIM_HDRS := $(wildcard $(PKG)/include/vcsched/*.hpp)

$(SHIM): $(SRC)/vcsched_b200.cpp $(SHIM_HDRS) include/vcs_gpu.h $(LIB)
	$(CXX) -O2 -std=c++20 -fPIC -shared -Wall -I$(PKG)/include -o $@ $(SRC)/vcsched_b200.cpp \
	    -L$(PKG) -lvcs_gpu -Wl,-rpath,'$$ORIGIN'

# the reference CLI's schedule / speedup subcommands over the shim (scheduler mdp-gpu added)
$(CLI): $(SRC)/vcsched_cli.cpp $(SHIM) $(SHIM_HDRS)
	$(CXX) -O2 -std=c++20 -Wall -I$(PKG)/include -o $@ $(SRC)/vcsched_cli.cpp \
	    -L$(PKG) -lvcsched_b200 -lvcs_gpu -Wl,-rpath,'$$ORIGIN'

$(ORACLE): oracle/vcs_oracle.c include/vcs_gpu.h
	$(CC) -O2 -std=gnu11 -fPIC -shared -ffp-contract=off -pthread -o $@ $< -lm

# The unmodified reference, compiled from its own sources where they lie (never copied), with
# the reference's Release flags (-O3 -DNDEBUG, no -march), plus the C shim of oracle/ref_capi.cpp.
# Linked against the system's shared libstdc++ (the one numpy/torch load): a toolchain wrapper that
# links libstdc++ statically made the reference's iostream parser crash inside such a process.
ref:
	@if [ -d $(REF)/core/src ]; then $(MAKE) --no-print-directory $(REFLIB) $(REF_SUITES); \
	 else echo "reference sources absent: using the prebuilt $(REFLIB) if present"; fi

$(REFLIB): oracle/ref_capi.cpp include/vcs_gpu.h
	@mkdir -p oracle/_ref
	$(REF_CXX) -std=c++20 -O3 -DNDEBUG -fPIC -shared -pthread -I$(REF)/core/include -I$(REF)/tests -I$(JSON_INC) \
	    -o $@ $(REF)/core/src/*.cpp oracle/ref_capi.cpp

# The reference's OWN solver test suites (doctest files compiled where they lie, unchanged),
# linked (a) against the reference library as the control and (b) against the B200 drop-in shim.
REF_TESTS  := $(REF)/tests/test_workload.cpp $(REF)/tests/test_greedy.cpp \
              $(REF)/tests/test_mdp.cpp $(REF)/tests/test_parallel.cpp
REF_SUITES := oracle/_ref/ref_suite_on_reference oracle/_ref/ref_suite_on_b200 \
              oracle/_ref/acceptance_on_b200

oracle/_ref/ref_suite_on_reference: tests/cpp/doctest.h tests/cpp/doctest_main.cpp
	@mkdir -p oracle/_ref
	$(CXX) -std=c++20 -O2 -pthread -Itests/cpp -I$(REF)/core/include -I$(REF)/tests -I$(JSON_INC) \
	    -DVCSCHED_DATA_DIR='"tests/golden"' -o $@ $(REF_TESTS) tests/cpp/doctest_main.cpp \
	    $(REF)/core/src/*.cpp

oracle/_ref/ref_suite_on_b200: tests/cpp/doctest.h tests/cpp/doctest_main.cpp $(SHIM) $(SHIM_HDRS)
	@mkdir -p oracle/_ref
	$(CXX) -std=c++20 -O2 -pthread -Itests/cpp -I$(PKG)/include -I$(REF)/tests \
	    -DVCSCHED_DATA_DIR='"tests/golden"' -o $@ $(REF_TESTS) tests/cpp/doctest_main.cpp \
	    -L$(PKG) -lvcsched_b200 -lvcs_gpu -Wl,-rpath,'$$ORIGIN/../../$(PKG)'

clean:
	rm -rf build $(LIB) $(SHIM) $(CLI) $(ORACLE) oracle/_ref

.PHONY: all ref clean

# The reference's acceptance suite (tests/acceptance.cpp, unchanged) against the drop-in shim.
# Its criteria 6-9 exercise the reference's DSRC simulator / metrics (out of scope for the B200
# path): those translation units are the reference's own sources, compiled where they lie.
REF_SIM := $(REF)/core/src/metrics.cpp $(REF)/core/src/sim.cpp $(REF)/core/src/channel.cpp
oracle/_ref/acceptance_on_b200: $(SHIM) $(SHIM_HDRS)
	@mkdir -p oracle/_ref
	$(CXX) -std=c++20 -O2 -pthread -I$(PKG)/include -I$(REF)/core/include -I$(REF)/tests \
	    -DVCSCHED_DATA_DIR='"tests/golden"' -o $@ $(REF)/tests/acceptance.cpp $(REF_SIM) \
	    -L$(PKG) -lvcsched_b200 -lvcs_gpu -Wl,-rpath,'$$ORIGIN/../../$(PKG)'
