#!/bin/bash
# GPU-box check: parity tests, smoke, bench, ncu launch list + full captures
# of the headline kernel and the other hot kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
if [ "${NCU:-1}" = "1" ]; then
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 5 --warmup 3 --no-extras > gpurun_out/ncu_bench_cfg2.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_bench_cfg2.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_bench.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_tile -s 3 -c 1 -o gpurun_out/prof_cfg2 -f python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
timeout 600 ncu --set full --clock-control none -k regex:"k_red|k_chain|k_gemm|k_tf32" -c 12 -o /tmp/prof_hot -f python scripts/hot_kernels.py > gpurun_out/ncu_hot.log 2>&1
echo "ncu hot rc=$?" >> gpurun_out/ncu_hot.log
ncu -i /tmp/prof_hot.ncu-rep --page raw --csv > gpurun_out/prof_hot_raw.csv 2>/dev/null
ncu -i /tmp/prof_hot.ncu-rep --page details --csv > gpurun_out/prof_hot_details.csv 2>/dev/null
fi
du -sh gpurun_out
