#!/bin/bash
# cloth HVP timings for tile sizes (variant libraries via MG_LIB)
cd paper_2509_00406_b200/csrc
build() { rm -rf build; make -j8 EXTRA="$2" OUT=/tmp/lib_$1.so >/dev/null 2>&1 || echo "build $1 failed"; }
build t64 "-DMG_TILE_ROWS=64 -DMG_TILE_VPT=3"
build t256 "-DMG_TILE_ROWS=256 -DMG_TILE_VPT=2"
build t128m6 "-DEV_TILE_MINB=6"
rm -rf build; make -j8 >/dev/null 2>&1
cd ../..
for i in 1 2; do
  for v in default t64 t256 t128m6; do
    lib=""; [ $v != default ] && lib=/tmp/lib_$v.so
    echo "$v $(MG_LIB=$lib MG_DEBUG_TILES=1 timeout 300 python bench.py --only --profile-call hvp --steps 30 2>&1 | grep -v '^edge tiles' | tail -1)"
  done
done
