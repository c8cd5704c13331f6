# K9e (sliced-ELL b = 1) + windowed K8 prefetch: tests, b = 1 timings, top-k segment sweep, launch list
set -x
O=gpurun_out/r02ac; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_prune.py -x -q > $O/tests.log 2>&1; echo "tests rc=$?"; tail -5 $O/tests.log
for segs in 0 16 32 64 148; do
timeout 600 python tools/stream_probe.py --batches 1 --topk-segs $segs > $O/b1_sell_segs$segs.jsonl 2> $O/b1_sell_segs$segs.err; echo "probe rc=$?"; head -1 $O/b1_sell_segs$segs.jsonl
done
timeout 600 python tools/stream_probe.py --batches 1 --single csr > $O/b1_csr.jsonl 2> $O/b1_csr.err; head -1 $O/b1_csr.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "k9s:b1/" --csv --log-file $O/launches_b1_sell.csv python tools/stream_probe.py --batches 1 --steps 3 > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
