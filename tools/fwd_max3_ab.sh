# Sequential A/B of the forward's row-max reduction: FMNMX3 (current tree) vs the previous 2-input form
# (git stash of the kernel is not available on the box, so the old form is rebuilt with SPT_FWD_MAX2).
for v in new old new old; do
  touch paper_2506_13996_b200/csrc/attention_tc.cu
  if [ $v = old ]; then SPT_EXTRA_DEFS=SPT_FWD_MAX2 python paper_2506_13996_b200/build.py > /dev/null; else python paper_2506_13996_b200/build.py > /dev/null; fi
  echo "max=$v"; python tools/attn_rank_bench.py 32768 32 8 | tail -1; python tools/attn_rank_bench.py 524288 4 1 | tail -1
done
