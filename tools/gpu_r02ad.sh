# few-rows histogram top-k + K9e: tests, b = 1 timings, launch list
set -x
O=gpurun_out/r02ad; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_prune.py -x -q > $O/tests.log 2>&1; echo "tests rc=$?"; tail -5 $O/tests.log
timeout 600 python tools/stream_probe.py --batches 1,8 > $O/b1_sell.jsonl 2> $O/b1_sell.err; echo "probe rc=$?"; head -2 $O/b1_sell.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "k9s:b1/" --csv --log-file $O/launches_b1_sell.csv python tools/stream_probe.py --batches 1 --steps 3 > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
