#!/bin/bash
# Full ncu capture of one mid-sequence decode step (step $STEP, default 35)
# of the benchmark batch (eager launches, tools/profile_run.py):
#   1) launch list -> index of the step's first kernel (k_embed_target)
#   2) ncu --set full over that step's kernels
set -e
STEP=${STEP:-35}
OUT=${OUT:-gpurun_out}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/step_list.csv \
    python tools/profile_run.py $PR_ARGS > /dev/null 2>&1
read SKIP COUNT < <(python - "$OUT/step_list.csv" "$STEP" <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
ki, mi = rows[h].index("Kernel Name"), rows[h].index("Metric Name")
names = [r[ki] for r in rows[h + 1:] if len(r) > mi and r[mi] == "gpu__time_duration.sum"]
starts = [i for i, n in enumerate(names) if "k_embed_target" in n]
s = int(sys.argv[2])
print(starts[s], starts[s + 1] - starts[s])
PY
)
echo "step $STEP: skip $SKIP count $COUNT"
ncu --set full --clock-control none -f -s $SKIP -c $COUNT -o /tmp/step_full \
    python tools/profile_run.py $PR_ARGS > $OUT/ncu_step.log 2>&1
ncu -i /tmp/step_full.ncu-rep --page raw --csv --metrics \
gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active,lts__t_bytes.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread \
    > $OUT/step_full_raw.csv
ncu -i /tmp/step_full.ncu-rep --page details > $OUT/step_full_details.txt 2>&1
ls -la /tmp/step_full.ncu-rep
echo done
