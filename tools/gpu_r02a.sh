set -x
mkdir -p gpurun_out/r02a
nvidia-smi > gpurun_out/r02a/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02a/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02a/gputest.log
timeout 900 python bench.py > gpurun_out/r02a/bench.json 2> gpurun_out/r02a/bench.err; echo "bench rc=$?"
FAST="--steps 2 --warmup 3 --no-sweep --no-parity --no-cpu-baseline --skip-e2e --no-offline-warmup"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "fsr:online/" --csv --log-file gpurun_out/r02a/launches_online.csv python bench.py $FAST > gpurun_out/r02a/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k9t_gemm --launch-skip 3 -c 1 -o gpurun_out/r02a/k9t_full python bench.py $FAST > gpurun_out/r02a/ncu_full.log 2>&1; echo "ncu full rc=$?"
