# A/B: _ab_head (a worktree of the base commit, built) vs the working tree
for i in 1 2; do
  echo "== base"; (cd _ab_head && python tools/attn_bench.py)
  echo "== new";  python tools/attn_bench.py
done
