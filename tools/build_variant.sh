#!/bin/bash
# Build a tuning variant of libs2attn.so with extra nvcc flags:
#   tools/build_variant.sh <name> "-DS2_DKV_NST=2 ..."
# -> paper_2407_17678_b200/variants/<name>/libs2attn.so, selected at run time
#    with S2ATTN_VARIANT=<name> (tuning experiments only).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1
mkdir -p "$ROOT/paper_2407_17678_b200/variants/$NAME"
make -s -j16 -C "$ROOT/paper_2407_17678_b200/csrc" "$ROOT/paper_2407_17678_b200/variants/$NAME/libs2attn.so" \
  OUT="$ROOT/paper_2407_17678_b200/variants/$NAME/libs2attn.so" BUILD="$ROOT/build/variant_$NAME" EXTRA_NVFLAGS="$2"
