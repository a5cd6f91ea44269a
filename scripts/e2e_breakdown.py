"""Time the e2e path of bench.py piece by piece (load / enumerate / free) for one config."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2401_05039_b200 import make_config, mbe_enumerate, mbe_free, mbe_load_csr  # noqa: E402
from paper_2401_05039_b200 import inputs as I  # noqa: E402

g = I.config_graph(sys.argv[1] if len(sys.argv) > 1 else "C5")
rp = torch.from_numpy(np.ascontiguousarray(g.row_ptr, dtype=np.uint64)).pin_memory().numpy()
ci = torch.from_numpy(np.ascontiguousarray(g.col_idx, dtype=np.uint32)).pin_memory().numpy()
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = mbe_load_csr(g.n1, g.n2, rp, ci)
    t1 = time.perf_counter()
    r = mbe_enumerate(h, make_config())
    t2 = time.perf_counter()
    mbe_free(h)
    t3 = time.perf_counter()
    print(f"load {1e3*(t1-t0):.1f} ms  enumerate {1e3*(t2-t1):.1f} ms (kernel {r.kernel_ms:.1f}, wall {r.wall_ms:.1f})"
          f"  free {1e3*(t3-t2):.1f} ms")
