python tools/config_ab.py mlp_tiles=0,1,4 --rounds 3 --group 12 > gpurun_out/r2d20_a.txt 2>&1; tail -1 gpurun_out/r2d20_a.txt
python tools/config_ab.py loss_tile=0,16384,4096 --rounds 3 --group 12 > gpurun_out/r2d20_b.txt 2>&1; tail -1 gpurun_out/r2d20_b.txt
