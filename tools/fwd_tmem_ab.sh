rm -f paper_2506_13996_b200/_build/attention_tc.cu.o
SPT_WATCHDOG=1 python -c "from paper_2506_13996_b200 import build as B; B.build()"
SPT_ATTN_FWD_TMEM=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k attention 2>&1 | tail -3
rm -f paper_2506_13996_b200/_build/attention_tc.cu.o
python -c "from paper_2506_13996_b200 import build as B; B.build()"
for M in 0 1 0 1; do echo "FWD_TMEM=$M"; SPT_ATTN_FWD_TMEM=$M python tools/attn_bench.py | sed -n 1p; SPT_ATTN_FWD_TMEM=$M python tools/attn_rank_bench.py 262144 4 1 | cut -c1-50; done
