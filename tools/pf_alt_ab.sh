# (Experiment record: the ELLM_PF_ALT build was measured with this script and then reverted,
# DESIGN.md §5 f4; the knob no longer exists in the sources.)
# f4: alternating exponential phases of the two Q tiles' softmax warps (ELLM_PF_ALT) A/B on one box,
# three alternating repetitions of tools/prefill_bench.py. usage: bash tools/pf_alt_ab.sh
python -m paper_2506_15155_b200.build > /dev/null 2>&1
for rep in 1 2 3; do for alt in 0 1; do
  echo "== ELLM_PF_ALT=$alt rep $rep"; ELLM_PF_ALT=$alt timeout 300 python tools/prefill_bench.py 2>&1 | grep TFLOP
done; done
