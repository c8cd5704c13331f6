# round-2 GPU job b: K2 vertex-order probe at C3, compute-sanitizer passes, fp64 C2 bench line
set -x
O=gpurun_out/r02b; mkdir -p $O
timeout 900 python tools/k2_order_probe.py > $O/k2_order.jsonl 2> $O/k2_order.err; echo "k2 probe rc=$?"
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_prune.py -x -q > $O/memcheck_prune.log 2>&1; echo "memcheck prune rc=$?"
timeout 900 $CS --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_tc.py -x -q -k "auto and not 20000" > $O/racecheck_tc.log 2>&1; echo "racecheck tc rc=$?"
timeout 900 $CS --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_tc.py -x -q -k "auto and not 20000" > $O/synccheck_tc.log 2>&1; echo "synccheck tc rc=$?"
timeout 900 $CS --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_prune.py -x -q -k "test_tc_small_and_odd_batches" > $O/racecheck_k9t.log 2>&1; echo "racecheck k9t rc=$?"
timeout 900 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_parity_c1.py -x -q > $O/memcheck_c1.log 2>&1; echo "memcheck c1 rc=$?"
timeout 900 python bench.py --config C2 --dtype float64 --no-sweep --steps 5 > $O/bench_c2_f64.json 2> $O/bench_c2_f64.err; echo "bench c2 f64 rc=$?"
