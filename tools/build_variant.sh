#!/bin/bash
# Build a tuning variant of the extension into build_variants/<name>/libapax_b200.so
# (the product .so is untouched).  Usage: tools/build_variant.sh <name> "-DKNOB=V ..."
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; DEFS=$2
OUT=$ROOT/build_variants/$NAME
mkdir -p $OUT/build
make -s -j8 -C $ROOT/paper_1303_4994_b200/csrc OUT=$OUT/libapax_b200.so BUILD=$OUT/build EXTRA="$DEFS"
