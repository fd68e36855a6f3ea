#!/bin/bash
# Builds liborx.so from git revision $1 into build/ab/liborx_$2.so (A/B timing:
# ORX_LIB_PATH=build/ab/liborx_$2.so python bench.py ...).
set -e
rev=$1; tag=$2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
git -C "$root" archive "$rev" paper_2506_13695_b200/csrc include | tar -x -C "$tmp"
mkdir -p "$root/build/ab"
make -C "$tmp/paper_2506_13695_b200/csrc" -j8 OUT="$root/build/ab/liborx_$tag.so" OBJDIR="$tmp/obj" > /dev/null
rm -rf "$tmp"
echo "$root/build/ab/liborx_$tag.so"
