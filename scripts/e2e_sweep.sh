#!/bin/bash
# A/B of the cfg2 e2e pipeline shape: result slabs by rows or by columns,
# 8/16/32 slabs (bench.py --no-extras; one JSON line each).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for split in cols rows; do
  for ch in 2 4 8 16; do
    echo -n "$split $ch " >> gpurun_out/e2e_sweep.txt
    TPG_E2E_SPLIT=$split TPG_E2E_CHUNKS=$ch timeout 300 python bench.py --steps 40 --warmup 5 --no-extras 2>>gpurun_out/e2e_sweep.err \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['e2e'])" >> gpurun_out/e2e_sweep.txt
  done
done
cat gpurun_out/e2e_sweep.txt
