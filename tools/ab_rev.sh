#!/bin/bash
# Build libxscatgpu.so of a git revision into build_ab/<name>/ (A/B against the
# working tree): tools/ab_rev.sh <rev> <name> [extra nvcc defines]
set -e
rev=$1; name=$2; shift 2
root=$(pwd)
tmp=$(mktemp -d)
git worktree add -q --detach $tmp $rev
make -C $tmp -j16 lib OBJDIR=$root/build_ab/$name/obj LIBDIR=$root/build_ab/$name NVEXTRA="$*" > $root/build_ab/$name.log 2>&1
git worktree remove --force $tmp
rm -rf build_ab/$name/obj
echo build_ab/$name/libxscatgpu.so
