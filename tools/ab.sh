# A/B: bench in the repo (B) vs the HEAD worktree under _ab_head (A), alternating
for i in 1 2; do
  for side in A B; do
    if [ $side = A ]; then d=_ab_head; else d=.; fi
    (cd $d && timeout 240 python bench.py --steps 9 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$side', d['value'], d['config']['value_single_stream'])")
  done
done
