#!/bin/bash
# Dirichlet row kernel occupancy variants (FV_MINB) on icosphere(9)
cd paper_2509_00406_b200/csrc
build() { rm -rf build; make -j8 EXTRA="$2" OUT=/tmp/lib_$1.so >/dev/null 2>&1 || echo "build $1 failed"; }
build m8 "-DFV_MINB=8"
build m5 "-DFV_MINB=5"
rm -rf build; make -j8 >/dev/null 2>&1
cd ../..
for v in default m8 m5; do
  lib=""; [ $v != default ] && lib=/tmp/lib_$v.so
  MG_LIB=$lib timeout 300 python tools/bench_configs.py --configs dirichlet --sub 9 --steps 10 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$v', d['call'], round(d['kernel_ms'],4))"
done
