"""Timing of the BRGEMM TPP on tcgen05 (K11): the cfg-2 composition as one
grouped launch per variant and one large brgemm() (bench.py's extra)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2104_05755_b200 as tpp  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
print(json.dumps(bench.brgemm_variants(torch, tpp, dev, g, 1681.7)))
