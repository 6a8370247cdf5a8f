#!/bin/bash
# Build an experimental libpdst variant from a patched copy of csrc/.
# usage: [NVCC_DEFS='-DPDST_TRACE'] scripts/build_variant.sh NAME 'sed-expression'|patch.py [file]   -> exp/libpdst_NAME.so
set -e
NAME=$1; EXPR=$2; FILE=${3:-pdst_operator.cu}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
mkdir -p "$TMP/pkg" && cp -r "$ROOT/paper_2603_28706_b200/csrc" "$TMP/pkg/csrc"
mkdir -p "$TMP/include" && cp "$ROOT/include/pdst.h" "$TMP/include/"
if [[ "$EXPR" == *.py ]]; then python3 "$EXPR" "$TMP/pkg/csrc/$FILE"; else sed -i "$EXPR" "$TMP/pkg/csrc/$FILE"; fi
mkdir -p "$ROOT/exp"
cd "$TMP/pkg/csrc"
nvcc $NVCC_DEFS -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -rdc=true -Xcompiler -fPIC -Xptxas -v -shared \
  -o "$ROOT/exp/libpdst_$NAME.so" pdst_operator.cu pdst_vector.cu pdst_krylov.cu pdst_patch.cu pdst_timediag.cu pdst_coarse.cu \
  pdst_mg.cu pdst_manufactured.cu pdst_strip.cu pdst_th.cu pdst_capi.cu -lcudart -ldl > "$ROOT/exp/build_$NAME.log" 2>&1 || { tail -5 "$ROOT/exp/build_$NAME.log"; exit 1; }
grep -A2 "k_jacobianILi2" "$ROOT/exp/build_$NAME.log" | grep -E "spill|registers" || true
rm -rf "$TMP"
