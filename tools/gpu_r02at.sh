# K8 prologue (y in shared memory, warp-scan prefix, w prefetch) + rank-by-counting top-k: tests and b = 1 timings
set -x
O=gpurun_out/r02at; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_prune.py tests/test_gpu_tc.py tests/test_gpu_parity_c1.py -x -q > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
for D in 0.01 0.02; do
timeout 600 python tools/stream_probe.py --batches 1,8 --density $D > $O/b1_d$D.jsonl 2> $O/b1_d$D.err; echo "d=$D"; head -2 $O/b1_d$D.jsonl | cut -c1-260
done
