"""GPU probe (tool): `maximum` of signed zeros through gevo_exec_once."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(HERE), os.path.dirname(os.path.dirname(HERE))]
from paper_2310_10211_b200 import _lib, dialect  # noqa: E402
from test_gpu_parity import run_once  # noqa: E402

for n in (6, 600):
    fn = dialect.parse_function(f"""func @f(%a: tensor<{n}xf32>, %b: tensor<{n}xf32>) -> tensor<{n}xf32> {{
  %0 = maximum %a, %b : tensor<{n}xf32>
  return %0 : tensor<{n}xf32>
}}""")
    a = np.resize(np.array([np.nan, 1.0, np.nan, -np.inf, -0.0, 0.0]), n)
    b = np.resize(np.array([1.0, np.nan, np.nan, np.inf, 0.0, -0.0]), n)
    ctx = _lib.Context(0)
    (got,), = run_once(ctx, [fn], [[a, b]])
    ctx.close()
    print(n, "device", got[:6].tolist(), "numpy", np.maximum(a, b)[:6].tolist(),
          "signbits dev", np.signbit(got[:6]).tolist(), "np", np.signbit(np.maximum(a, b)[:6]).tolist())
