"""One prefill_attention config for profiling: python tools/prefill_one.py B ctx n_q [T]"""
import sys

sys.path.insert(0, ".")
from tools.prefill_bench import run  # noqa: E402

B, ctx, nq = (int(x) for x in sys.argv[1:4])
T = int(sys.argv[4]) if len(sys.argv) > 4 else 16
run(B, ctx, nq, T=T, iters=2)
