#!/bin/bash
# A/B (experiment switch TPG_GEMM_GROUP, removed after it -- profiles/r02s_gemm_traffic_vs_cublas.md):
# raster group height (256-row tiles per group) of the CTA-pair gemm:
# burst TFLOP/s (bench extras cfg4) and DRAM / L2 bytes per launch (ncu).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for gsz in 8 16 32 4 8; do
  echo -n "group=$gsz " >> gpurun_out/gemm_group.txt
  TPG_GEMM_GROUP=$gsz timeout 300 python scripts/extras_probe.py cfg4 >> gpurun_out/gemm_group.txt 2>> gpurun_out/gemm_group.err
done
for gsz in 8 16 32; do
  TPG_GEMM_GROUP=$gsz timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -k regex:k_gemm_sm100_pair -c 4 --csv --log-file gpurun_out/gemm_group_ncu_$gsz.csv python scripts/gemm_traffic_probe.py > /dev/null 2>&1
done
