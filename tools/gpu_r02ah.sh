# K9e long rows (8 rows x 128 entries per warp step, side stream): tests, threshold sweep at 2% / 5%, bench sweep with settle
set -x
O=gpurun_out/r02ah; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_kernels.py -x -q -k "sell or topk or b1 or u16" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
for L in 128 256 512; do
for D in 0.02 0.05; do
timeout 600 python tools/stream_probe.py --batches 1 --sell-long $L --density $D > $O/b1_L${L}_d$D.jsonl 2> $O/b1_L${L}_d$D.err; echo "L=$L d=$D"; head -1 $O/b1_L${L}_d$D.jsonl
done; done
timeout 1200 python bench.py --no-cpu-baseline --no-parity > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
