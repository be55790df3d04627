#!/bin/bash
# Build libpasd_b200.so with extra -D flags into build/<name>.so (timing
# experiments: select it with PASD_B200_LIB=build/<name>.so).
#   tools/build_variant.sh name -DPASD_P2_FAST=0 ...
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_1712_09999_b200/csrc"
mkdir -p ../../build
make -s NVFLAGS_EXTRA="$*" OUT=../../build/$name.so
