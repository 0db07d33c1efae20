#!/bin/bash
# Config 5 on a GPU box (under gpurun): launch list, then application replay of
# one iteration's big kernels (kernel replay cannot save / restore the 64 GiB
# working set), reduced on the box by tools/ncu_summary.py.
OUT=${OUT:-gpurun_out/prof}
TAG=${TAG:-r02}
mkdir -p $OUT
args="--config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
python bench.py $args > $OUT/plain_c5.json 2>&1 || exit 1
kpi=$(python -c "import json;print(json.loads(open('$OUT/plain_c5.json').read().strip().splitlines()[-1])['config']['iteration_graph_kernels'])")
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file $OUT/launches_c5.csv python bench.py $args > /dev/null 2>&1
ncu --replay-mode application --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
    -k regex:"gemm_xm1|gemm_streamk|k_stencil_tma|k_update_norm|k_bb_cols" -s ${SKIP:-14} -c ${COUNT:-14} \
    --csv --log-file $OUT/app_c5.csv python bench.py $args > $OUT/ncu_app_c5.log 2>&1
python tools/ncu_summary.py --launches $OUT/launches_c5.csv --app-csv $OUT/app_c5.csv \
    --config 5 --tag $TAG --kpi $kpi --outdir $OUT
