# Attention A/B: parity tests + timing of the current build, then forward poly-exp2 fraction variants.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "attention or layer or fullsize" > gpurun_out/attn_tests.log 2>&1; tail -3 gpurun_out/attn_tests.log
python tools/attn_bench.py > gpurun_out/attn_ab.txt 2>&1; echo "poly4:" ; cat gpurun_out/attn_ab.txt
for E in 0 2 3 8; do
  rm -f paper_2506_13996_b200/_build/attention_tc.cu.o
  SPT_EXTRA_DEFS=SPT_FWD_POLY_EVERY=$E python -c "from paper_2506_13996_b200 import build as B; B.build()"
  echo "poly every $E:"; python tools/attn_bench.py 2>&1 | head -2
done
