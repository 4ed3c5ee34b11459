for X in NONE SPT_EXP_HALF_KV; do
  rm -f paper_2506_13996_b200/_build/attention_tc.cu.o
  SPT_EXTRA_DEFS=$X python -c "from paper_2506_13996_b200 import build as B; B.build()"
  echo "$X:"
  timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,l1tex__m_xbar2l1tex_read_bytes.sum.per_second --clock-control none -k regex:dq_tc -c 1 --csv python tools/attn_bench.py 2>/dev/null | grep dq_tc | awk -F'","' '{print $(NF-2), $NF}'
  timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:dq_tc -c 1 --csv python tools/attn_rank_bench.py 131072 4 1 2>/dev/null | grep dq_tc | awk -F'","' '{print $(NF-2), $NF}'
done
