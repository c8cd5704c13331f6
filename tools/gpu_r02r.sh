# kNN block timing at C3 + 2-rank functional bench (gloo, one GPU) at C1 + new kernel test
set -x
O=gpurun_out/r02r; mkdir -p $O
timeout 600 python tools/knn_probe.py > $O/knn_probe.json 2> $O/knn_probe.err; echo "knn probe rc=$?"
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k u16 > $O/tests.log 2>&1; echo "tests rc=$?"
FSR_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --config C1 --steps 3 --warmup 3 --no-sweep --no-cpu-baseline --batch 256 > $O/bench_2rank_gloo_c1.json 2> $O/bench_2rank.err; echo "2-rank rc=$?"
