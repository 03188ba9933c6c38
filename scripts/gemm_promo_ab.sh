#!/bin/bash
# A/B (experiment switch TPG_GEMM_PROMO, removed after it): L2 promotion of the
# gemm operand tensor maps: burst
# TFLOP/s (extras cfg4) and DRAM / L2 bytes per launch (ncu).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for pr in 2 0 1 2 0 1; do
  echo -n "promo=$pr " >> gpurun_out/gemm_promo.txt
  TPG_GEMM_PROMO=$pr timeout 300 python scripts/extras_probe.py cfg4 >> gpurun_out/gemm_promo.txt 2>> gpurun_out/gemm_promo.err
done
for pr in 0 1 2; do
  TPG_GEMM_PROMO=$pr timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -k regex:k_gemm_sm100_pair -c 4 --csv --log-file gpurun_out/gemm_promo_ncu_$pr.csv python scripts/gemm_traffic_probe.py > /dev/null 2>&1
done
