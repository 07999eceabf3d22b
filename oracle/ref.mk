# Builds the REFERENCE ITSELF (unmodified sources under /root/reference/proj) against
# the header-only Eigen / doctest shims in oracle/ref_shim/ — TEST INFRASTRUCTURE
# (SURVEY.md §8(c) Route A).  Outputs go only to oracle/_ref/ (git-ignored; the built
# files travel to the GPU box, the reference sources do not).  The reference's own
# CMake build is not used: it needs find_package(Eigen3), absent from this image.
#
#   make -f oracle/ref.mk            # libauxmc_ref.so + the C bridge + unit/acceptance tests
#   oracle/_ref/auxmc_tests          # the reference's doctest suite on the shim
#   oracle/_ref/acceptance           # the reference's acceptance criteria
REF     ?= /root/reference/proj
HERE    := $(dir $(lastword $(MAKEFILE_LIST)))
OUT     := $(HERE)_ref
JSONDIR ?= $(firstword $(wildcard /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann) \
                       $(wildcard $(HERE)ref_shim/nlohmann))
CXX     ?= g++
# -ffp-contract=off: no FMA contraction (x86-64 baseline has no FMA anyway), so the
# reference's arithmetic is evaluated as written.
CXXFLAGS ?= -O2 -g0 -DNDEBUG -fPIC -std=c++20 -ffp-contract=off -w
INC     := -I$(HERE)ref_shim -I$(REF)/include -I$(JSONDIR)

LIB_SRCS := gauss lgssm pit target auxk fkpg bench/models bench/grid_hmm bench/diagnostics bench/config bench/runner
LIB_OBJS := $(patsubst %,$(OUT)/obj/%.o,$(LIB_SRCS))
TEST_SRCS := test_main test_rng test_gauss test_lgssm test_scan test_pit test_target_auxk test_fkpg test_bench
TEST_OBJS := $(patsubst %,$(OUT)/obj/tests/%.o,$(TEST_SRCS))
SHIM_DEPS := $(wildcard $(HERE)ref_shim/Eigen/*) $(HERE)ref_shim/doctest.h

all: $(OUT)/libauxmc_ref.so $(OUT)/libref_bridge.so $(OUT)/auxmc_tests $(OUT)/acceptance

$(OUT)/obj/%.o: $(REF)/src/%.cpp $(SHIM_DEPS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) $(INC) -c $< -o $@

$(OUT)/obj/tests/%.o: $(REF)/tests/%.cpp $(SHIM_DEPS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) $(INC) -I$(REF)/tests -c $< -o $@

$(OUT)/libauxmc_ref.so: $(LIB_OBJS)
	$(CXX) -shared -o $@ $(LIB_OBJS) -lpthread

# C bridge (oracle/ref_bridge.cpp, our code): flat extern "C" entry points over the
# reference's C++ API for the Python parity tests and the CPU baseline.  Self-contained:
# the reference objects and a private static libstdc++ (symbols hidden), so the C++
# runtime exported by other extension modules of the host Python process (numpy's core
# module re-exports libstdc++ type_info and locale symbols) cannot interpose on its
# iostreams and exceptions.
$(OUT)/libref_bridge.so: $(HERE)ref_bridge.cpp $(LIB_OBJS) $(SHIM_DEPS)
	$(CXX) $(CXXFLAGS) $(INC) -I$(REF)/tests -shared -static-libstdc++ -static-libgcc \
	  -Wl,--exclude-libs,ALL -o $@ $< $(LIB_OBJS) -lpthread

$(OUT)/auxmc_tests: $(TEST_OBJS) $(OUT)/libauxmc_ref.so
	$(CXX) -o $@ $(TEST_OBJS) -L$(OUT) -lauxmc_ref -Wl,-rpath,'$$ORIGIN' -lpthread

$(OUT)/acceptance: $(REF)/tests/acceptance.cpp $(OUT)/libauxmc_ref.so $(SHIM_DEPS)
	$(CXX) $(CXXFLAGS) $(INC) -I$(REF)/tests -o $@ $< -L$(OUT) -lauxmc_ref -Wl,-rpath,'$$ORIGIN' -lpthread

clean:
	rm -rf $(OUT)
.PHONY: all clean
