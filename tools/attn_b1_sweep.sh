# batch-1 self-attention: heads per CTA and staging cap (tools/attn_bench.py, B=1)
for k in 1 5; do for hg in 2 4 8; do for cap in 48 64; do
  echo "K=$k HG=$hg CAP=$cap"; B=1 K=$k SKB_ATTN_HG=$hg SKB_ATTN_CAP=$cap python tools/attn_bench.py
done; done; done
