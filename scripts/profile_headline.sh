cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 5 --warmup 3 --no-extras > gpurun_out/ncu_l1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 > gpurun_out/ncu_l2.log 2>&1
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none -k regex:k_tile_tma -c 40 --csv --log-file gpurun_out/cfg2_steady_dram.csv python bench.py --steps 20 --warmup 3 --no-extras > gpurun_out/ncu_l3.log 2>&1
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_tile_tma -c 20 --csv --log-file gpurun_out/cfg2_cold_dram.csv python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/ncu_l4.log 2>&1
timeout 300 ncu --set full --cache-control none --clock-control none --import-source on -k regex:k_tile_tma -s 12 -c 1 -o gpurun_out/prof_cfg2_steady -f python bench.py --steps 20 --warmup 3 --no-extras > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/prof_cfg2_steady.ncu-rep --page details --csv > gpurun_out/prof_cfg2_steady_details.csv 2>/dev/null
ncu -i gpurun_out/prof_cfg2_steady.ncu-rep --page raw --csv > gpurun_out/prof_cfg2_steady_raw.csv 2>/dev/null
