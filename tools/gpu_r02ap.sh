# K9e gather depth 4 / 8 / 16 at C3 1% / 2%
set -x
O=gpurun_out/r02ap; mkdir -p $O
for D in 4 8 16; do
FSR_K9E_DEPTH=$D timeout 600 python tools/stream_probe.py --batches 1 --density 0.02 > $O/b1_depth$D.jsonl 2> $O/b1_depth$D.err; echo "depth=$D"; head -1 $O/b1_depth$D.jsonl | cut -c1-260
done
