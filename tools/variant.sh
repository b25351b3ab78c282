#!/bin/bash
# Build an A/B variant of libdtans.so into variants/NAME/ (git-ignored, but
# it travels to the GPU box).  SRC = a git revision, or "wt" for the working
# tree; EXTRA = extra nvcc flags (e.g. -DDTANS_PEND_NP=1).
#   tools/variant.sh NAME SRC [EXTRA...]
set -e
cd "$(dirname "$0")/.."
NAME=$1; SRC=$2; shift 2
D=/tmp/variant_src_$NAME
rm -rf $D && mkdir -p $D
if [ "$SRC" = wt ]; then
  tar -c --exclude=./variants --exclude=./gpurun_out --exclude=./build --exclude=./.git --exclude=./baseline . | tar -x -C $D
else
  git archive $SRC | tar -x -C $D
fi
mkdir -p variants/$NAME
make -s -C $D/paper_2603_01915_b200/csrc OUT=$PWD/variants/$NAME/libdtans.so BUILD=$D/build EXTRA="$*" 2>&1 | grep -iE "error|spill stores" | grep -v " 0 bytes spill" | head -5 || true
ls -la variants/$NAME/libdtans.so
