rm -f paper_2506_13996_b200/_build/attention_tc.cu.o
SPT_EXTRA_DEFS=SPT_DQ_PROF python -c "from paper_2506_13996_b200 import build as B; B.build()"
python tools/dq_prof.py
python tools/dq_prof.py 262144 4 1
