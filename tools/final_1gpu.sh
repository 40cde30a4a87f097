#!/bin/bash
# Round-end check on one B200, as the driver runs it: the GPU test suite, smoke(), then
# the N = 1 measurement set (tools/measure_r2.sh, with its ncu passes)
set -u
O=${O:-gpurun_out/final1}
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -n 2 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke OK')" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 $O/smoke.log
O=$O bash tools/measure_r2.sh
