import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from tests import test_gpu_layer as T
from oracle import sptrain_oracle as O
for cfg, shape in ((T.QWENISH, T.QWENISH_SHAPE), (O.LayerConfig(320, 4, 2, 128, 640, 1024), T.S.ModelShape(320, 4, 2, 128, 640, 1024)),
                   (O.LayerConfig(256, 4, 1, 128, 640, 1024), T.S.ModelShape(256, 4, 1, 128, 640, 1024)),
                   (O.LayerConfig(320, 4, 1, 80, 640, 1024), T.S.ModelShape(320, 4, 1, 80, 640, 1024))):
    try:
        r = T._run(1, 1024, cfg=cfg, shape=shape)
    except Exception as e:
        print(cfg, "ERR", e); continue
    print(cfg, "loss", r["loss"], {k: bool(np.isnan(v).any()) for k, v in r["grads"].items()}, "dx nan", bool(np.isnan(r["dx"]).any()))
