# Compile-time A/B of the 128-key forward's P hand-off parts (SPT_FWD2_NPART 2 vs 4), sequential builds.
for np in 2 4 2 4; do
  touch paper_2506_13996_b200/csrc/attention_tc.cu
  SPT_EXTRA_DEFS=SPT_FWD2_NPART=$np python paper_2506_13996_b200/build.py > /dev/null
  echo "NPART=$np"; python tools/attn_rank_bench.py 32768 32 8 | tail -1; python tools/attn_rank_bench.py 524288 4 1 | tail -1
done
