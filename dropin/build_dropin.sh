#!/usr/bin/env bash
# Drop-in proof build: the reference's own unit tests (proj/tests/*.cpp except
# test_io.cpp), compiled unmodified from where they lie, linked against
#   - dropin/ptychodd_ops_cuda.cpp    (fft.hpp, forward.hpp, stagm.hpp over the
#                                     C-ABI; replaces proj/src/fft.cpp,
#                                     forward.cpp, stagm.cpp)
#   - dropin/ptychodd_solver_cuda.cpp (NonblindSolver, BlindSolver over the
#                                     C-ABI; replaces proj/src/solver.cpp,
#                                     blind.cpp)
#   - the reference's remaining sources (field, scan, ddplan, simulate,
#     metrics: data structures, integer planning, test-data generation and
#     the metrics, which now call the GPU operators), and
#   - paper_2011_00162_b200/libptychodd_cuda.so.
# The test framework header is dropin/doctest.h (doctest is not in the image).
# Also the reference's acceptance program (proj/tests/acceptance.cpp, the
# paper's criteria 1-6) and its pybind module (proj/python/bindings.cpp ->
# _ptychodd) linked the same way.
# Output: dropin/_build/ptychodd_dropin_{tests,acceptance} (git-ignored; they
# travel to the GPU box with the snapshot).
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
CXX="g++ -std=c++20 -O2 -DNDEBUG -I$ref/include -I$here -I$repo/include"
objs=()
for s in field scan ddplan simulate metrics; do
  $CXX -c "$ref/src/$s.cpp" -o "$out/ref_$s.o" &
  objs+=("$out/ref_$s.o")
done
for t in test_main test_field_fft test_forward test_stagm test_ddplan test_simulate test_metrics test_solver test_blind; do
  $CXX -c "$ref/tests/$t.cpp" -o "$out/$t.o" &
  objs+=("$out/$t.o")
done
$CXX -c "$here/ptychodd_solver_cuda.cpp" -o "$out/ptychodd_solver_cuda.o" &
$CXX -c "$here/ptychodd_ops_cuda.cpp" -o "$out/ptychodd_ops_cuda.o" &
wait
objs+=("$out/ptychodd_solver_cuda.o" "$out/ptychodd_ops_cuda.o")
$CXX -c "$ref/tests/acceptance.cpp" -o "$out/acceptance.o"
lib="$repo/paper_2011_00162_b200"
link() { g++ -o "$1" "${@:2}" -L"$lib" -lptychodd_cuda -Wl,-rpath,'$ORIGIN/../../paper_2011_00162_b200' -lpthread; }
link "$out/ptychodd_dropin_tests" "${objs[@]}"
# the reference's acceptance program (paper criteria 1-6) on the same library
lib_objs=()
for o in "${objs[@]}"; do case "$o" in */test_*.o) ;; *) lib_objs+=("$o") ;; esac; done
link "$out/ptychodd_dropin_acceptance" "${lib_objs[@]}" "$out/acceptance.o"
# the reference's pybind front-end (proj/python/bindings.cpp, unmodified): the
# Python reconstruct / reconstruct_blind entry points routed to the GPU library
pyinc="$(python3 -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
pybind="$(python3 -c 'import pybind11; print(pybind11.get_include())')"
ext="$(python3 -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
PYCXX="g++ -std=c++20 -O2 -DNDEBUG -fPIC -fvisibility=hidden -I$ref/include -I$here -I$repo/include -I$pyinc -I$pybind"
pyobjs=()
for s in field scan ddplan simulate metrics; do
  $PYCXX -c "$ref/src/$s.cpp" -o "$out/py_ref_$s.o" & pyobjs+=("$out/py_ref_$s.o")
done
$PYCXX -c "$here/ptychodd_solver_cuda.cpp" -o "$out/py_solver.o" & pyobjs+=("$out/py_solver.o")
$PYCXX -c "$here/ptychodd_ops_cuda.cpp" -o "$out/py_ops.o" & pyobjs+=("$out/py_ops.o")
$PYCXX -c "$ref/python/bindings.cpp" -o "$out/py_bindings.o" & pyobjs+=("$out/py_bindings.o")
wait
g++ -shared -o "$out/_ptychodd$ext" "${pyobjs[@]}" -L"$lib" -lptychodd_cuda \
  -Wl,-rpath,'$ORIGIN/../../paper_2011_00162_b200' -lpthread
rm -f "$out"/*.o
echo "built $out/ptychodd_dropin_tests $out/ptychodd_dropin_acceptance $out/_ptychodd$ext"
