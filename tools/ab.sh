# A/B timing: bench in this tree (B) vs a baseline worktree under _ab_head (A),
# alternating, two rounds.  Create / update the baseline with
#   git worktree add -f _ab_head <commit>   (or: git -C _ab_head checkout --detach <commit>)
#   (cd _ab_head && python -c "from paper_2207_05851_b200 import build; build.build(force=True)")
# _ab_head is git-ignored but travels with gpurun.
for i in 1 2; do
  for side in A B; do
    if [ $side = A ]; then d=_ab_head; else d=.; fi
    (cd $d && timeout 240 python bench.py --steps 9 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$side', d['value'], d['config']['value_single_stream'])")
  done
done
