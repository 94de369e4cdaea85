"""Golden TBST1 checkpoint + logs.csv written by the REFERENCE itself (build container only):

    python tests/golden/make_tbst1.py

Writes tests/golden/beastpipe_mlp.tbst1 (beastpipe.pipeline.checkpoint of a small
init_params MLP with non-zero heads, version 7) and tests/golden/beastpipe_logs.csv
(beastpipe.pipeline.MetricsWriter with two records).
"""
import os
import shutil
import sys
import tempfile
from dataclasses import replace

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from beastpipe import model as bm  # noqa: E402
from beastpipe import pipeline as bp  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
p = bm.init_params(obs_dim=10, num_actions=3, hidden=4, seed=5)
rng = np.random.default_rng(6)
p = replace(p, Wp=rng.normal(size=p.Wp.shape).astype(np.float32),
            bv=np.array([0.25], np.float32), version=7)
bp.checkpoint(p, os.path.join(HERE, "beastpipe_mlp.tbst1"))
d = tempfile.mkdtemp()
w = bp.MetricsWriter(d)
for rec in (bp.MetricsRecord(1, 160, 1.5, -0.25, 3.125, -0.0125, 2.8625, 1234.5678),
            bp.MetricsRecord(2, 320, float("nan"), 0.5, 1.0, -0.01, 1.49, 99.999)):
    w.append(rec)
w.close()
shutil.copy(os.path.join(d, "logs.csv"), os.path.join(HERE, "beastpipe_logs.csv"))
print("ok")
