#!/bin/bash
# headline timings for row-block sizes (variant libraries via MG_LIB)
cd paper_2509_00406_b200/csrc
for rb in 32 128; do
  rm -rf build; make -j8 EXTRA="-DMG_ROW_BLOCK=$rb" OUT=/tmp/lib_rb$rb.so >/dev/null 2>&1 || echo "build $rb failed"
done
rm -rf build; make -j8 >/dev/null 2>&1
cd ../..
for i in 1 2; do
  for rb in default 32 128; do
    lib=""; [ $rb != default ] && lib=/tmp/lib_rb$rb.so
    echo "rb=$rb $(MG_LIB=$lib timeout 300 python bench.py --only --profile-call psd --steps 30 2>/dev/null | tail -1)"
  done
done
