#!/bin/bash
# compute-sanitizer memcheck over this round's new device paths: the drop-in
# plugin (managed storage, lazy-cast fusion, flags take, descriptor
# transfers), the sharded device finish (tpg_shard_pack / unpack, NCCL
# world 1) and the standalone layer's error modes / stream bookkeeping.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 \
  python -m pytest -q -x -p no:cacheprovider -m gpu tests/test_plugin.py tests/test_gpu_sharded.py \
  tests/test_gpu_modes.py -k "not full_size" > gpurun_out/sanitize_r02_memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/sanitize_r02_memcheck.log
tail -5 gpurun_out/sanitize_r02_memcheck.log
