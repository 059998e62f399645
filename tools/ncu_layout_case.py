"""ncu driver: one large device layout conversion (DLT, vl=4) of a 2D storage array."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_08825_b200 import transpose as tr  # noqa: E402
from paper_2103_08825_b200.grid import GridBuffer, Layout  # noqa: E402

rows, unp, hu = 8192, 8192, 2
like = GridBuffer(np.zeros((1, 1)), (rows - 2, unp), 1, unp, unp, Layout.DLT, 4)
src = torch.rand(rows, unp + 2 * hu, dtype=torch.float64, device="cuda")
dst = torch.empty_like(src)
for to in (True, False):
    tr.convert_device(src, dst, like, to)
torch.cuda.synchronize()
print("layout conversions done")
