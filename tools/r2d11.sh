python tools/fwd_det_check.py 4096 8 2 2.5 11,21,13,23
timeout 900 python tools/attn_fwd_ab.py 13,11 32768:32:8 524288:4:1 --rounds 3 2>&1 | grep -v "O rel"
timeout 900 python tools/attn_fwd_ab.py 13,11 32768:32:8 524288:4:1 --rounds 3 --lib=ab_old/libsptrain_b200.so 2>&1 | grep -v "O rel"
