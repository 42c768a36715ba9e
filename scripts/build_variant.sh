#!/usr/bin/env bash
# Build an alternative libhcb (tuning experiments): scripts/build_variant.sh TAG "-DFOO=1 -DBAR=2"
# -> paper_1912_01478_b200/libhcb_TAG.so (load with HCB_LIB=libhcb_TAG.so)
set -e
cd "$(dirname "$0")/../paper_1912_01478_b200/csrc"
make -s -j"$(nproc)" VAR="$1" VFLAGS="$2"
