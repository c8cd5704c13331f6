# launch list of the offline decomposition at C3 (NVTX fsr:offline)
set -x
O=gpurun_out/r02as; mkdir -p $O
FAST="--steps 2 --warmup 3 --no-sweep --no-parity --no-cpu-baseline --skip-e2e --no-offline-warmup"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "fsr:offline/" --csv --log-file $O/launches_offline.csv python bench.py $FAST > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
python tools/summarize_launches.py $O/launches_offline.csv | head -40
