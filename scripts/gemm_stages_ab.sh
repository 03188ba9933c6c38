#!/bin/bash
# A/B of the CTA-pair gemm ring depth (P_STAGES 6 = product, 5, 4; libs built
# by scripts/build_ab.py from temporary revisions), burst cfg4 numbers from
# bench.extras, interleaved, same box.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/gemm_stages_ab.txt
for i in 1 2; do
  for lib in base st5 st4; do
    echo -n "$lib " >> $out
    TIDEPOOL_GPU_LIB=ab_libs/lib_$lib.so timeout 300 python -c "
import sys; sys.path.insert(0, '.')
import bench, paper_1810_08723_b200 as tp
from paper_1810_08723_b200 import _native
r = bench.extras(tp, tp.gpu(0), _native.lib(), only={'cfg4'})
print({k: v.get('TFLOP/s') for k, v in r.items()})" 2>>gpurun_out/gemm_stages_ab.err >> $out
  done
done
cat $out
