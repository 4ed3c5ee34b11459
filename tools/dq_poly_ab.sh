for E in 0 4 8 2; do
  rm -f paper_2506_13996_b200/_build/attention_tc.cu.o
  SPT_EXTRA_DEFS=SPT_DQ_POLY_EVERY=$E python -c "from paper_2506_13996_b200 import build as B; B.build()"
  echo "dq poly every $E:"; python tools/attn_bench.py 2>&1 | sed -n 2p
done
