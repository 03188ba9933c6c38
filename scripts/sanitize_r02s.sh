#!/bin/bash
# compute-sanitizer over the r02s device / host-path changes: the TMA-fed
# cfg2 tile kernel (memcheck + racecheck + synccheck on the tile tests, which
# cover every reversal, Y mode and tile shape) and the drop-in's C entry
# paths / block pool (memcheck on the plugin tests).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --error-exitcode 9 \
    python -m pytest -q -x -p no:cacheprovider -m gpu tests/test_gpu_tile.py \
    -k "reversals and INT16 or tile_shapes or cfg2_shape" > gpurun_out/sanitize_r02s_tile_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_r02s_tile_$tool.log
  tail -3 gpurun_out/sanitize_r02s_tile_$tool.log
done
timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 \
  python -m pytest -q -x -p no:cacheprovider -m gpu tests/test_plugin.py -k "not full_size and not threads" > gpurun_out/sanitize_r02s_plugin.log 2>&1
echo "plugin memcheck rc=$?" >> gpurun_out/sanitize_r02s_plugin.log
tail -3 gpurun_out/sanitize_r02s_plugin.log
