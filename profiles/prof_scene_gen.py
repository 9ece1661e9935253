"""16,384 C3 obstacle courses (k_gen) for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_10247_b200 import world as wd  # noqa: E402

for i in range(3):
    wd.gen_obstacle_courses(100 + i, 16384, [0.0, 0.0, 1.2], [8.0, 0.0, 1.5], 32 / 48.0, device="cuda", check=False)
torch.cuda.synchronize()
print("ok")
