for hg in 2 4 8; do for cap in 32 48 64; do echo "HG=$hg CAP=$cap"; SKB_ATTN_HG=$hg SKB_ATTN_CAP=$cap python tools/attn_bench.py; done; done
