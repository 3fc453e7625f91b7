#!/bin/bash
# A/B build of libxscatgpu.so with extra nvcc defines, into build_ab/<name>/ (the
# product lib/ is never touched); run with XSCAT_LIB=build_ab/<name>/libxscatgpu.so.
#   tools/ab.sh <name> "-DXSW_INNER=2 ..."
set -e
name=$1; shift
make -j16 lib OBJDIR=build_ab/$name/obj LIBDIR=build_ab/$name NVEXTRA="$*" > build_ab/$name.log 2>&1 || { mkdir -p build_ab; make -j16 lib OBJDIR=build_ab/$name/obj LIBDIR=build_ab/$name NVEXTRA="$*"; }
rm -rf build_ab/$name/obj
echo build_ab/$name/libxscatgpu.so
