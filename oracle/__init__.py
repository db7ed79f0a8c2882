"""CPU oracle for the NCHW[x]c conv hot path -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference (`neoplan`, /root/reference/pkg/src)
algorithms on the north_star path.  Each function cites the reference
file:line it restates.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` leg may import this
package, and only as the checker or as the timed CPU baseline; the product
package (paper_1809_02697_b200) never imports it and has no CPU fallback.

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
golden vectors produced by running the reference itself
(``tests/golden/make_golden.py``, committed with the fixtures), plus the
reference's own known-answer properties (tests/test_layout.py:74-117,
tests/test_kernels.py:71-83, 175-186).
"""

from .ops import (add, batchnorm, concat, conv2d, dense, flatten, nhwc_to_nchw,
                  pack_kcrs, pack_nchw, pool2d, relu, rel_err, retile_nchw,
                  softmax, transform, unpack_kcrs, unpack_nchw)
from .graph_exec import execute_reference

__all__ = ["add", "batchnorm", "concat", "conv2d", "dense", "flatten",
           "nhwc_to_nchw", "pack_kcrs", "pack_nchw", "pool2d", "relu",
           "rel_err", "retile_nchw", "softmax", "transform", "unpack_kcrs",
           "unpack_nchw", "execute_reference"]
