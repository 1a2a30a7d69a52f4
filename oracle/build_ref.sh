#!/usr/bin/env bash
# Builds oracle/_ref/libfgsref.so (TEST INFRASTRUCTURE ONLY): the reference's
# own hot-path sources, compiled UNCHANGED from where they lie under
# /root/reference/proj/src, against the shim headers in oracle/shim (the
# Eigen3 / FFTW3 stand-ins; neither library is in this image), plus the C
# entry layer oracle/ref_capi.cpp.  Flags follow the reference's default
# Release build (proj/CMakeLists.txt:8-10,36: -O3 -DNDEBUG, no FMA on x86-64
# without -march, i.e. -ffp-contract=off).  Output goes only to oracle/_ref/
# (git-ignored; it travels to the GPU box with the snapshot).  Nothing is
# copied out of /root/reference.
set -euo pipefail
here="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
ref="${FGS_REFERENCE:-/root/reference/proj}"
if [ ! -d "$ref/src" ]; then
  echo "build_ref: $ref not present; keeping any prebuilt oracle/_ref" >&2
  exit 0
fi
mkdir -p "$here/_ref"
g++ -std=c++20 -O3 -DNDEBUG -ffp-contract=off -fPIC -shared -w \
    -I "$here/shim" -I "$ref/include" \
    "$ref/src/nfft.cpp" "$ref/src/kernels.cpp" "$ref/src/fastsum.cpp" "$ref/src/graphop.cpp" \
    "$ref/src/spectral.cpp" "$here/ref_capi.cpp" \
    -o "$here/_ref/libfgsref.so"
echo "$here/_ref/libfgsref.so"
