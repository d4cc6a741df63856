#!/bin/bash
# Build fused-kernel tuning variants into build/variants/<name>/ (experiments
# only; the product library is paper_1910_00572_b200/libgridloc_b200.so).
set -e
cd "$(dirname "$0")/../paper_1910_00572_b200/csrc"
for v in "$@"; do
  name=${v%%:*}; flags=${v#*:}
  mkdir -p ../../build/variants/$name
  make -s -j8 OUT=../../build/variants/$name/libgridloc_b200.so OBJDIR=../../build/variants/$name/obj \
       EXTRA_NVFLAGS="-DGL_EXPERIMENT_ENV $flags" EXTRA_CXXFLAGS="-DGL_EXPERIMENT_ENV"
done
