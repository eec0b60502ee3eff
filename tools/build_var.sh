#!/bin/bash
# usage: tools/build_var.sh NAME "-DKNOB=1 ..." -- builds build/var_NAME/libbsg.so with extra nvcc flags
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
make -s -C "$ROOT/paper_2106_06161_b200/csrc" -j16 EXTRA="$2" OUTDIR="$ROOT/build/var_$1" OBJDIR="$ROOT/build/obj_var_$1" >/dev/null
echo "built build/var_$1/libbsg.so ($2)"
