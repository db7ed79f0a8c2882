import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from test_gpu_fp8 import _conv, _check_close_e4m3
import numpy as np
for case, tile in [((2, 64, 32, 32, 128, 3, 3, 1, 1, 64, 128, False, True), None),
                   ((2, 64, 32, 32, 128, 3, 3, 1, 1, 64, 128, False, True), {"tile_n": 128, "weight_stationary": 1}),
                   ((2, 64, 32, 32, 128, 3, 3, 1, 1, 64, 64, False, True), {"tile_n": 64}),
                   ((2, 64, 32, 32, 64, 3, 3, 1, 1, 64, 64, False, True), None),
                   ((2, 64, 20, 20, 128, 3, 3, 1, 1, 64, 128, False, True), None),
                   ((1, 64, 56, 56, 128, 3, 3, 1, 1, 64, 128, False, True), None)]:
    got, ref = _conv(*case, tile=tile)
    d = got != ref
    print(case, tile, "mismatch frac", d.mean())
