#!/usr/bin/env bash
# Drop-in proof build: the reference's own unit tests for the solver layer
# (proj/tests/test_solver.cpp, test_blind.cpp), compiled unmodified from where
# they lie, linked against
#   - the reference's non-solver sources (field, fft, scan, forward, stagm,
#     ddplan, simulate, metrics: test-data generation and the transparent
#     reference ADMM the tests compare against; fft via oracle/fftw_shim),
#   - dropin/ptychodd_solver_cuda.cpp, which defines NonblindSolver and
#     BlindSolver (replacing proj/src/solver.cpp and blind.cpp) over
#     include/ptychodd_cuda.h, and
#   - paper_2011_00162_b200/libptychodd_cuda.so.
# The test framework header is dropin/doctest.h (doctest is not in the image).
# Output: dropin/_build/ptychodd_dropin_tests (git-ignored; travels to the GPU
# box with the snapshot).  Run there:  dropin/_build/ptychodd_dropin_tests
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
repo="$(dirname "$here")"
ref="${PDD_REFERENCE:-/root/reference}/proj"
out="$here/_build"
if [ ! -d "$ref/src" ]; then
  echo "build_dropin.sh: reference sources not found at $ref (skipping)" >&2
  exit 0
fi
mkdir -p "$out"
CXX="g++ -std=c++20 -O2 -DNDEBUG -I$ref/include -I$repo/oracle/fftw_shim -I$here -I$repo/include"
objs=()
for s in field fft scan forward stagm ddplan simulate metrics; do
  $CXX -c "$ref/src/$s.cpp" -o "$out/ref_$s.o" &
  objs+=("$out/ref_$s.o")
done
for t in test_main test_solver test_blind; do
  $CXX -c "$ref/tests/$t.cpp" -o "$out/$t.o" &
  objs+=("$out/$t.o")
done
$CXX -c "$repo/oracle/fftw_shim/fftw_shim.cpp" -o "$out/fftw_shim.o" &
$CXX -c "$here/ptychodd_solver_cuda.cpp" -o "$out/ptychodd_solver_cuda.o" &
wait
objs+=("$out/fftw_shim.o" "$out/ptychodd_solver_cuda.o")
lib="$repo/paper_2011_00162_b200"
g++ -o "$out/ptychodd_dropin_tests" "${objs[@]}" -L"$lib" -lptychodd_cuda -Wl,-rpath,'$ORIGIN/../../paper_2011_00162_b200' \
  -lpthread
rm -f "$out"/*.o
echo "built $out/ptychodd_dropin_tests"
