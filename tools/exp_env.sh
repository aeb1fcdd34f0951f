# usage: bash tools/exp_env.sh "ENV=.. ENV2=.." ...   (one bench per argument, 3 streams)
for cfg in "$@"; do
  tag=$(echo "$cfg" | tr ' =/' '_-_')
  env $cfg timeout 240 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/exp_$tag.log 2>&1
  echo "[$cfg] rc=$? $(tail -1 gpurun_out/exp_$tag.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"].get("value_single_stream"), d["batch1_latency"]["beam5"]["p50_ms"])' 2>&1 | tail -1)"
done
