for E in 0 8 4 3; do
  rm -f paper_2506_13996_b200/_build/attention_tc.cu.o
  SPT_EXTRA_DEFS=SPT_FWD_POLY_EVERY=$E python -c "from paper_2506_13996_b200 import build as B; B.build()"
  echo "poly every $E:"; python tools/attn_bench.py 2>&1 | head -1
done
