rm -f paper_2506_13996_b200/_build/attention_tc.cu.o
SPT_WATCHDOG=1 python -c "from paper_2506_13996_b200 import build as B; B.build()"
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k attention 2>&1 | tail -2
SPT_ATTN_FWD_TMEM=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "attention_fwd_bwd" 2>&1 | tail -1
rm -f paper_2506_13996_b200/_build/attention_tc.cu.o
python -c "from paper_2506_13996_b200 import build as B; B.build()"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
python tools/attn_bench.py | head -2
