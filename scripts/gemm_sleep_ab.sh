#!/bin/bash
# A/B: epilogue accumulator-wait back-off (TPG_GEMM_EPI_SLEEP ns) vs spinning,
# sustained cfg4 gemms with SM clock / power (scripts/gemm_vs_cublas.py).
# (The TPG_GEMM_EPI_SLEEP switch existed only for this A/B; it was removed after it
# showed no effect -- profiles/r02s_gemm_epilogue_backoff_ab.txt.)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for ns in 0 500 2000 0 500 2000; do
  echo -n "epi_sleep=$ns " >> gpurun_out/gemm_sleep_ab.txt
  TPG_GEMM_EPI_SLEEP=$ns timeout 300 python -c "
import sys; sys.path.insert(0, 'scripts'); import gemm_vs_cublas as g
print(g.sustained('ours'))" >> gpurun_out/gemm_sleep_ab.txt 2>> gpurun_out/gemm_sleep_ab.err
done
cat gpurun_out/gemm_sleep_ab.txt
