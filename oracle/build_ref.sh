#!/usr/bin/env bash
# ORACLE TEST INFRASTRUCTURE — builds the reference CPU path from its own,
# unmodified sources where they lie (/root/reference/proj/src), plus our
# FFTW-API shim (oracle/fftw_shim) and the extern "C" test wrapper
# (oracle/ref_capi.cpp), into oracle/_ref/libptychodd_ref.so.
#
# Flags follow the reference's Release default (proj/CMakeLists.txt:6-8:
# -O3 -DNDEBUG, C++20, no -march).  io.cpp (PTYA/JSON/CSV/PNG) compiles
# against the image's zlib and the nlohmann/json 3.11.3 header shipped in the
# venv (cudnn_frontend/thirdparty); it makes the reference's own PTYA files
# and dataset directories for the PTYA-streaming and CLI parity tests.  Output
# goes only to oracle/_ref/ (git-ignored; it travels to the GPU box).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
ref="${PDD_REFERENCE:-/root/reference}/proj"
out="$here/_ref"
if [ ! -d "$ref/src" ]; then
  echo "build_ref.sh: reference sources not found at $ref (skipping)" >&2
  exit 0
fi
mkdir -p "$out"
json_dir="${PDD_NLOHMANN:-$(python - <<'PY'
import glob, os, sys
c = glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "include", "cudnn_frontend",
                           "thirdparty", "nlohmann", "json.hpp"))
print(os.path.dirname(c[0]) if c else "")
PY
)}"
srcs=(field fft scan forward stagm ddplan solver blind simulate metrics)
if [ -n "$json_dir" ] && [ -f /usr/include/zlib.h ]; then srcs+=(io); fi
objs=()
for s in "${srcs[@]}"; do
  o="$out/ref_$s.o"
  g++ -std=c++20 -O3 -DNDEBUG -fPIC -I"$ref/include" -I"$here/fftw_shim" ${json_dir:+-I"$json_dir"} \
    -c "$ref/src/$s.cpp" -o "$o"
  objs+=("$o")
done
g++ -std=c++20 -O3 -DNDEBUG -fPIC -c "$here/fftw_shim/fftw_shim.cpp" -o "$out/fftw_shim.o"
io_def=""
[[ " ${srcs[*]} " == *" io "* ]] && io_def="-DREF_HAVE_IO"
g++ -std=c++20 -O3 -DNDEBUG -fPIC -I"$ref/include" -I"$here/fftw_shim" ${json_dir:+-I"$json_dir"} $io_def \
  -c "$here/ref_capi.cpp" -o "$out/ref_capi.o"
g++ -shared -o "$out/libptychodd_ref.so" "${objs[@]}" "$out/fftw_shim.o" "$out/ref_capi.o" -lpthread ${io_def:+-lz}
rm -f "$out"/*.o
echo "built $out/libptychodd_ref.so"
