# ncu of the K9t finish / threshold / sample kernels at C3 b=1024; bench with adaptive kNN certification
set -x
O=gpurun_out/r02j; mkdir -p $O
FAST="--steps 2 --warmup 3 --no-sweep --no-parity --no-cpu-baseline --skip-e2e --no-offline-warmup"
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "fsr:online/" -k regex:"k9t_finish|k9t_threshold" -c 2 -o $O/k9t_sel python bench.py $FAST > $O/ncu_sel.log 2>&1; echo "ncu rc=$?"
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
