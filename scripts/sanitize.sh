#!/bin/bash
# compute-sanitizer runs of parity subsets on the GPU box (race
# detection / memory checking).  Summaries go to gpurun_out/sanitize_*.log.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool memcheck --leak-check no --error-exitcode 9 \
  python -m pytest -q -x -p no:cacheprovider tests/test_gpu_golden.py tests/test_gpu_chain.py \
  "tests/test_gpu_reduce.py::test_reduce_nan_first_and_inner" "tests/test_gpu_gemm.py::test_gemm_mn_major_operands" \
  "tests/test_gpu_reduce.py::test_column_chunking_regimes" \
  > gpurun_out/sanitize_memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/sanitize_memcheck.log
timeout 900 $CS --tool racecheck --error-exitcode 9 \
  python -m pytest -q -x -p no:cacheprovider "tests/test_gpu_reduce.py::test_reduce_nan_first_and_inner" \
  "tests/test_gpu_tile.py::test_cfg2_shape_all_sources" "tests/test_gpu_reduce.py::test_column_chunking_regimes" \
  > gpurun_out/sanitize_racecheck.log 2>&1
echo "racecheck rc=$?" >> gpurun_out/sanitize_racecheck.log
timeout 600 $CS --tool synccheck --error-exitcode 9 \
  python -m pytest -q -x -p no:cacheprovider "tests/test_gpu_reduce.py::test_reduce_full_large_f64" \
  > gpurun_out/sanitize_synccheck.log 2>&1
echo "synccheck rc=$?" >> gpurun_out/sanitize_synccheck.log
