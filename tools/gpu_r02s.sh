# kNN with libfsr top-k + concatenated bf16x3: probe, input tests, C2 certified graph, bench inputs
set -x
O=gpurun_out/r02s; mkdir -p $O
timeout 600 python tools/knn_probe.py > $O/knn_probe.json 2> $O/knn_probe.err; echo "knn probe rc=$?"
timeout 1200 python -m pytest tests/test_gpu_inputs.py tests/test_gpu_parity_c2.py -x -q -k "bf16 or bound or graph or queries" > $O/tests.log 2>&1; echo "tests rc=$?"
timeout 900 python bench.py --steps 5 --no-sweep --no-parity --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
