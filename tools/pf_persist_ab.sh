# (Experiment record: the persistent-grid build (ELLM_PF_PERSIST) was measured with this script
# and then reverted, DESIGN.md §5 f4; the knob no longer exists in the sources.)
# f4 persistent grid A/B on one box: the in-tree build with its grid heuristic, the same build with
# one CTA per item (ELLM_PF_PERSIST=0) and always persistent (=1), and $ELLM_LIB_PATH_B (the
# previous kernel, one CTA per item). Three alternating repetitions of tools/prefill_bench.py.
for rep in 1 2 3; do
  echo "== heuristic rep $rep"; timeout 300 python tools/prefill_bench.py 2>&1 | grep TFLOP
  echo "== PERSIST=0 rep $rep"; ELLM_PF_PERSIST=0 timeout 300 python tools/prefill_bench.py 2>&1 | grep TFLOP
  echo "== PERSIST=1 rep $rep"; ELLM_PF_PERSIST=1 timeout 300 python tools/prefill_bench.py 2>&1 | grep TFLOP
  echo "== previous kernel rep $rep"; ELLM_LIB_PATH=$ELLM_LIB_PATH_B timeout 300 python tools/prefill_bench.py 2>&1 | grep TFLOP
done
