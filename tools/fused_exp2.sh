for X in "SPT_EXP_NO_DQORDER,SPT_EXP_NO_DQWAIT" "SPT_EXP_NO_DQORDER"; do
  rm -f paper_2506_13996_b200/_build/attention_tc.cu.o
  SPT_EXTRA_DEFS=$X python -c "from paper_2506_13996_b200 import build as B; B.build()"
  echo "$X:"; SPT_ATTN_BWD=fused timeout 120 python tools/attn_bench.py 2>&1 | tail -n +2 | head -1
done
