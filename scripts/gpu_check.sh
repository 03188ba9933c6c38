#!/bin/bash
# GPU-box check: parity tests, smoke, bench, ncu launch list + one full capture.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 180 python -m pytest tests/test_gpu_gemm.py -q -rf -x > gpurun_out/pytest_gemm.log 2>&1
echo "gemm rc=$?" >> gpurun_out/pytest_gemm.log
timeout 900 python -m pytest tests -m gpu -q -rf --deselect tests/test_gpu_gemm.py > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
if [ "${NCU:-1}" = "1" ]; then
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_bench.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_tile -s 3 -c 1 -o gpurun_out/prof_cfg2 -f python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
fi
if [ "${NCU_RED:-1}" = "1" ]; then
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_red_rows -s 2 -c 1 -o gpurun_out/prof_red -f python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, paper_1810_08723_b200 as tp
X = tp.from_numpy(np.asfortranarray(np.random.default_rng(5).random((8192, 8192))))
for _ in range(4): tp.reduce('sum', X, axes=(0,))
tp.gpu(0).synchronize()
" > gpurun_out/ncu_red.log 2>&1
echo "ncu red rc=$?" >> gpurun_out/ncu_red.log
fi
