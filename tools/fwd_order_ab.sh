for X in 0 1 0 1; do
  rm -f paper_2506_13996_b200/_build/attention_tc.cu.o
  SPT_EXTRA_DEFS=SPT_FWD_ORDER=$X python -c "from paper_2506_13996_b200 import build as B; B.build()"
  echo "order $X:"; python tools/attn_bench.py 2>&1 | head -1; python tools/attn_rank_bench.py 131072 4 1 | cut -c1-60
done
rm -f paper_2506_13996_b200/_build/attention_tc.cu.o
SPT_EXTRA_DEFS=SPT_FWD_ORDER=1 python -c "from paper_2506_13996_b200 import build as B; B.build()"
timeout 600 python -m pytest tests -m gpu -q -x -k "attention" 2>&1 | tail -1
