#!/bin/bash
# One profiling pass on a GPU box (run under gpurun): bench lines, ncu launch
# lists and --set full captures of one iteration's kernels per config, reduced
# ON THE BOX to text summaries under $OUT (raw .ncu-rep files are deleted:
# gpurun copies back at most 64 MiB).  Each ncu command runs only after the
# same bench command exited 0 without ncu.
OUT=${OUT:-gpurun_out/prof}
TAG=${TAG:-r02}
mkdir -p $OUT
for c in ${CONFIGS:-2 3 4}; do
  args="--config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
  python bench.py $args > $OUT/plain_c$c.json 2>&1 || continue
  kpi=$(python -c "import json;print(json.loads(open('$OUT/plain_c$c.json').read().strip().splitlines()[-1])['config']['iteration_graph_kernels'])")
  ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
      --log-file $OUT/launches_c$c.csv python bench.py $args > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on \
      -k regex:"gemm_|k_stencil_tma|k_update_norm|k_bb_cols" -s ${SKIP:-12} -c ${COUNT:-6} \
      -o $OUT/full_c$c python bench.py $args > $OUT/ncu_full_c$c.log 2>&1
  python tools/ncu_summary.py --launches $OUT/launches_c$c.csv --full $OUT/full_c$c.ncu-rep \
      --config $c --tag $TAG --kpi $kpi --outdir $OUT > /dev/null 2>&1
  for k in gemm_xm1_staged gemm_xm_staged "gemm_streamk<pcal::GemmCfg<(int)128, (int)128, (int)2, (int)4, (int)3, (int)1" k_stencil_tma gemm_streamk; do
    python tools/ncu_stalls.py $OUT/full_c$c.ncu-rep "$k" 20 > "$OUT/stalls_c${c}_$(echo $k | tr -c 'a-z0-9_' '_' | cut -c1-40).txt" 2>&1
  done
  rm -f $OUT/full_c$c.ncu-rep
done
du -sh $OUT
