# Compile-time A/B of the 128-key forward's K/V ring depth (SPT_FWD2_NSL 4 vs 5), sequential builds.
for n in 4 5 4 5; do
  touch paper_2506_13996_b200/csrc/attention_tc.cu
  SPT_EXTRA_DEFS=SPT_FWD2_NSL=$n python paper_2506_13996_b200/build.py > /dev/null
  echo "NSL=$n"; python tools/attn_rank_bench.py 32768 32 8 | tail -1; python tools/attn_rank_bench.py 524288 4 1 | tail -1
done
