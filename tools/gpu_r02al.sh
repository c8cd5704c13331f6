# K9e small batches, persistent CTAs + co-running passes: tests, timings vs the CSR narrow kernels
set -x
O=gpurun_out/r02al; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_kernels.py -x -q -k "sell" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
for D in 0.01 0.02; do
timeout 900 python tools/stream_probe.py --batches 2,4,8,16,32,64 --density $D > $O/small_d$D.jsonl 2> $O/small_d$D.err; echo "sell d=$D rc=$?"; head -6 $O/small_d$D.jsonl | cut -c1-250
timeout 900 python tools/stream_probe.py --batches 8,16,32,64 --density $D --single csr > $O/small_csr_d$D.jsonl 2> $O/small_csr_d$D.err; echo "csr d=$D rc=$?"; head -4 $O/small_csr_d$D.jsonl | cut -c1-250
done
