# usage: bash tools/exp_env.sh "ENV=.. ENV2=.." ...   (one bench per argument, 3 streams)
for cfg in "$@"; do
  tag=$(echo "$cfg" | tr ' =/' '_-_')
  env $cfg timeout 300 python bench.py --steps ${STEPS:-6} --warmup 3 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/exp_$tag.log 2>&1
  echo "[$cfg] rc=$? $(tail -1 gpurun_out/exp_$tag.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"].get("value_single_stream"), d["roofline"]["ms_per_decode_step_gemms"])' 2>&1 | tail -1)"
done
