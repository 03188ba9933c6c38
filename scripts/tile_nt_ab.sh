#!/bin/bash
# A/B of k_tile_tma tiles per CTA iteration: 2 tiles by 16 warps (HEAD build)
# vs one tile by 8 warps (ab_libs/lib_nt1.so, scripts/build_ab.py).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/tile_nt_ab.txt
for i in 1 2 3; do
  for lib in "" ab_libs/lib_nt1.so; do
    echo -n "lib=${lib:-HEAD} " >> $out
    env ${lib:+TIDEPOOL_GPU_LIB=$lib} timeout 300 python bench.py --steps 40 --warmup 5 --no-extras 2>>gpurun_out/tile_nt_ab.err \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], r['achieved'], r['frac'], d['ms_per_step'])" >> $out
    echo -n "   u8 " >> $out
    env ${lib:+TIDEPOOL_GPU_LIB=$lib} timeout 300 python scripts/cfg2_u8_probe.py 2>>gpurun_out/tile_nt_ab.err | tail -1 >> $out
  done
done
cat $out
