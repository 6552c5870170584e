"""Time the full->band stage alone (kernel classes) on a random skew matrix of order n.
python tools/f2b_time.py 32768   (env SKEWEIG_PANEL_G=.. to experiment)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1912_04062_b200 as sk  # noqa: E402
import skewgen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
A0 = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
skewgen.random_skew_lower_device(A0, n, n, torch.cuda.current_stream().cuda_stream)
ctx = sk.Context()
ctx.set_profiling(True)
for rep in range(2):
    A = A0.clone()
    sk.reduce_to_band(A, ctx=ctx)
    torch.cuda.synchronize()
    st = ctx.kernel_stats()
print(f"n={n} G={os.environ.get('SKEWEIG_PANEL_G', 'auto')} " +
      " ".join(f"{k}={v[0]:.1f}" for k, v in st.items() if v[0] > 0.5), flush=True)
