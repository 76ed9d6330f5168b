#!/bin/bash
# unclamped spring HVP: staged tiles vs row-kernel variants (prefetch depth x occupancy)
cd paper_2509_00406_b200/csrc
build() { rm -rf build; make -j8 EXTRA="$2" OUT=/tmp/lib_$1.so >/dev/null 2>&1 || echo "build $1 failed"; }
build m6t512 "-DEV_HVP_MAXI=6 -DEV_HVP_THREADS=512"
build m6t640 "-DEV_HVP_MAXI=6 -DEV_HVP_THREADS=640"
build m4t512 "-DEV_HVP_MAXI=4 -DEV_HVP_THREADS=512"
rm -rf build; make -j8 >/dev/null 2>&1
cd ../..
for i in 1 2; do
  echo "tiles $(timeout 300 python bench.py --only --profile-call hvp --steps 30 2>/dev/null | tail -1)"
  for v in m6t512 m6t640 m4t512; do
    echo "$v $(MG_EDGE_TILES=0 MG_LIB=/tmp/lib_$v.so timeout 300 python bench.py --only --profile-call hvp --steps 30 2>/dev/null | tail -1)"
  done
done
