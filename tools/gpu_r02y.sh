# K9t 2-SM (cta_group::2) opt-in: guarded correctness first, then bench A/B
set -x
O=gpurun_out/r02y; mkdir -p $O
FSR_K9T_CLUSTER=42 timeout 240 python -m pytest tests/test_gpu_prune.py -x -q -k "identical_to_unpruned and tc" > $O/t1.log 2>&1; echo "t1 rc=$?"
if grep -q "passed" $O/t1.log && ! grep -q "failed" $O/t1.log; then
  FSR_K9T_CLUSTER=42 timeout 600 python -m pytest tests/test_gpu_prune.py -x -q > $O/tests42.log 2>&1; echo "tests rc=$?"
  FSR_K9T_CLUSTER=42 timeout 900 python bench.py --no-sweep --no-cpu-baseline > $O/bench42.json 2> $O/bench42.err; echo "bench42 rc=$?"
  timeout 900 python bench.py --no-sweep --no-cpu-baseline > $O/bench22.json 2> $O/bench22.err; echo "bench22 rc=$?"
fi
