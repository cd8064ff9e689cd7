#!/bin/bash
# Build libffb200.so with extra nvcc flags into <repo>/libffb200_<name>.so
# (same-box A/B of compile-time variants).  usage: build_variant.sh name "-DFOO ..."
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
D=$(mktemp -d)
mkdir -p $D/pkg $D/include
cp -r $ROOT/paper_2505_22758_b200/csrc $ROOT/paper_2505_22758_b200/Makefile $D/pkg/
cp -r $ROOT/include/* $D/include/
make -C $D/pkg -j16 EXTRA="$2" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
cp $D/pkg/libffb200.so $ROOT/libffb200_$1.so
rm -rf $D
echo "built libffb200_$1.so ($2)"
