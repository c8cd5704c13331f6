# K9e small batches (2 / 4 queries per pass): tests, timings b in {1, 2, 4, 8, 16, 32, 64} at 1% / 2%
set -x
O=gpurun_out/r02ak; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_prune.py tests/test_gpu_tc.py -x -q > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
for D in 0.01 0.02; do
timeout 900 python tools/stream_probe.py --batches 1,2,4,8,16,32,64 --density $D > $O/small_d$D.jsonl 2> $O/small_d$D.err; echo "d=$D rc=$?"; head -7 $O/small_d$D.jsonl | cut -c1-260
done
