#!/bin/bash
# A/B of the cfg2 e2e transfer scheme (bench.py TPG_E2E_ZC, an experiment switch
# removed after this A/B -- profiles/r02s_e2e_zero_copy_ab.md): copy-engine
# pipeline vs result stored by the kernel into pinned host memory vs
# everything zero-copy.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for zc in 0 1 2 0 1 2; do
  echo -n "zc=$zc " >> gpurun_out/e2e_zc.txt
  TPG_E2E_ZC=$zc timeout 300 python bench.py --steps 40 --warmup 5 --no-extras 2>>gpurun_out/e2e_zc.err \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['e2e'])" >> gpurun_out/e2e_zc.txt
done
cat gpurun_out/e2e_zc.txt
