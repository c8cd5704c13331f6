# K9s simple kernel: parity + C3 sweep (NB default, then NB=4)
set -x
O=gpurun_out/r02e; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_prune.py -x -q > $O/prune_tests.log 2>&1; echo "prune tests rc=$?"
timeout 900 python bench.py --steps 10 --no-parity --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
FSR_K9S_NB=4 timeout 900 python bench.py --steps 5 --no-parity --no-cpu-baseline --skip-e2e > $O/bench_nb4.json 2> $O/bench_nb4.err; echo "bench nb4 rc=$?"
