# adaptive long-row length: tests + b = 1 / 8 timings at 1 / 2 / 5%
set -x
O=gpurun_out/r02bi; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity_c1.py -x -q > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
for D in 0.01 0.02 0.05; do
timeout 600 python tools/stream_probe.py --batches 1,8 --density $D > $O/b_d$D.jsonl 2> $O/b_d$D.err; echo "d=$D"; head -2 $O/b_d$D.jsonl | cut -c1-250
done
