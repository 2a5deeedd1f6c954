#!/bin/bash
# Build the current csrc tree as a named library variant for kernel A/B runs:
#   bash scripts/build_variant.sh NAME    -> paper_2304_11165_b200/lib/variants/NAME.so
# Selected at run time with PD_LIB_VARIANT=NAME (paper_2304_11165_b200/_lib.py).
set -e
cd "$(dirname "$0")/../paper_2304_11165_b200/csrc"
make -s
mkdir -p ../lib/variants
cp ../lib/libporediff_b200.so ../lib/variants/$1.so
echo "built variant $1"
