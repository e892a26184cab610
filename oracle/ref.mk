# Builds the UNMODIFIED reference (/root/reference/proj) as a checker --
# TEST INFRASTRUCTURE ONLY.  Outputs go to oracle/_ref/ (git-ignored; the
# built files travel to the GPU box with the gpurun snapshot, the reference
# sources do not).  Sources are compiled where they lie; nothing is copied.
#
# The reference's CMake build needs Eigen3, libpng and a vendored doctest
# (proj/CMakeLists.txt:10,14-15), none of which exist in this image; the
# stand-ins under oracle/refshim/ provide the subset it uses (Eigen dense
# algebra, a libpng stub -- PNG I/O is out of scope -- and doctest-lite).
#
#   make -f oracle/ref.mk
#
# One build serves as checker and as the CPU baseline: the flags are the
# reference's own CMake Release configuration (CMakeLists.txt:6-8: -O3
# -DNDEBUG, no -march, so x86-64 SSE2 and no FMA contraction; the explicit
# -ffp-contract=off only documents that).
#
# Products:
#   _ref/libsplat_ref.so      splat_core (all 12 sources) + oracle/ref_capi.cpp
#   _ref/unit_tests           the reference's unit suite (tests/test_*.cpp)
#   _ref/acceptance_tests     the reference's acceptance criteria
REF ?= /root/reference/proj
CXX ?= g++
HERE := $(dir $(abspath $(lastword $(MAKEFILE_LIST))))
OUT ?= $(HERE)_ref
OPT ?= -O3 -DNDEBUG -ffp-contract=off
CXXFLAGS := -std=c++20 $(OPT) -fPIC -pthread -I$(REF)/include -I$(HERE)refshim -w

CORE := scene image scene_io render ssim residuals trust_region optimizer dataset config harness checks
TESTS := test_main test_dual test_geometry test_scene_io test_render test_residuals \
         test_trust_region test_optimizer test_harness
SHIM := $(wildcard $(HERE)refshim/Eigen/*) $(HERE)refshim/doctest.h $(HERE)refshim/png.h

CORE_O := $(patsubst %,$(OUT)/obj/%.o,$(CORE))
TEST_O := $(patsubst %,$(OUT)/obj/%.o,$(TESTS))

all: $(OUT)/libsplat_ref.so $(OUT)/unit_tests $(OUT)/acceptance_tests

$(OUT)/obj/%.o: $(REF)/src/%.cpp $(SHIM)
	@mkdir -p $(OUT)/obj
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OUT)/obj/%.o: $(REF)/tests/%.cpp $(SHIM)
	@mkdir -p $(OUT)/obj
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OUT)/obj/ref_capi.o: $(HERE)ref_capi.cpp $(HERE)ref_capi.h $(SHIM)
	@mkdir -p $(OUT)/obj
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OUT)/libsplat_ref.so: $(CORE_O) $(OUT)/obj/ref_capi.o
	$(CXX) -shared -pthread -o $@ $^ -lz

$(OUT)/unit_tests: $(TEST_O) $(CORE_O)
	$(CXX) -pthread -o $@ $^ -lz

$(OUT)/acceptance_tests: $(OUT)/obj/acceptance.o $(CORE_O)
	$(CXX) -pthread -o $@ $^ -lz

clean:
	rm -rf $(OUT)

.PHONY: all clean
