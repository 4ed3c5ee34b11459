mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "attention" 2>&1 | tail -1
for N in 10 8; do
  rm -f paper_2506_13996_b200/_build/attention_tc.cu.o
  SPT_EXTRA_DEFS=SPT_DQ_NSL=$N python -c "from paper_2506_13996_b200 import build as B; B.build()"
  echo "NSL $N:"; python tools/attn_bench.py 2>&1 | head -2
done
