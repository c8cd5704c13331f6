# GPU suite under the device-assertion build (FSR_DEBUG_CHECKS=1), standing in for compute-sanitizer
set -x
O=gpurun_out/r02bg; mkdir -p $O
FSR_DEBUG_CHECKS=1 timeout 900 python -m paper_1703_06935_b200.build --force > $O/build_debug.log 2>&1; echo "debug build rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -rs > $O/gputest_debugchecks.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_debugchecks.log 2>&1; echo "smoke rc=$?"
