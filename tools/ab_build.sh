#!/bin/bash
# Build library variants for an A/B run (here, before gpurun; *.so are
# git-ignored but travel with the snapshot). usage: bash tools/ab_build.sh "name:-DFLAG=.. -DFLAG2=.." ...
set -e
root=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$root/ab_libs"
for v in "$@"; do
  n=${v%%:*}; f=${v#*:}
  rm -rf /tmp/ab_build_$n; mkdir -p /tmp/ab_build_$n
  cp "$root"/paper_2509_00406_b200/csrc/*.cu "$root"/paper_2509_00406_b200/csrc/*.cuh "$root"/paper_2509_00406_b200/csrc/*.h "$root"/paper_2509_00406_b200/csrc/Makefile /tmp/ab_build_$n/
  mkdir -p /tmp/ab_include && cp "$root"/include/meshgrad_b200.h /tmp/ab_include/
  (cd /tmp/ab_build_$n && sed -i 's#../../include/meshgrad_b200.h#/tmp/ab_include/meshgrad_b200.h#' Makefile *.cuh *.cu 2>/dev/null; \
   make -j8 EXTRA="$f" OUT="$root/ab_libs/lib_$n.so" >/tmp/ab_build_$n.log 2>&1) &
done
wait
ls -la "$root/ab_libs"
