# K9e CTA size 128 / 256 / 512 / 1024 threads at C3 1% / 2%
set -x
O=gpurun_out/r02aw; mkdir -p $O
for T in 128 256 512 1024; do
for D in 0.01 0.02; do
FSR_K9E_THREADS=$T timeout 600 python tools/stream_probe.py --batches 1 --density $D > $O/b1_t${T}_d$D.jsonl 2> $O/b1_t${T}_d$D.err; echo "threads=$T d=$D"; head -1 $O/b1_t${T}_d$D.jsonl | cut -c1-260
done; done
