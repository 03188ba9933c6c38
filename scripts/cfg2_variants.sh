#!/bin/bash
# A/B of headline-kernel build variants (scripts/_variants/*/libtidepool_gpu.so)
# against the product library, same script, same box
for lib in product scripts/_variants/*/libtidepool_gpu.so; do
  if [ "$lib" = product ]; then unset TIDEPOOL_GPU_LIB; else export TIDEPOOL_GPU_LIB=$PWD/$lib; fi
  echo "== $lib"
  python scripts/cfg2_ceilings.py 2>&1 | grep -E "headline" | head -1
done
