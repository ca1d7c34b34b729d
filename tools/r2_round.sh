#!/bin/bash
# Round-2 checkpoint on one B200: smoke, full GPU test suite, then every measurement of
# tools/round_measure_r2.sh (bench line, configs, launch lists, ncu captures, projection).
set -u
o=gpurun_out/${TAG:-r2r}
mkdir -p $o
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $o/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --durations=25 > $o/gputest.log 2>&1
TAG=${TAG:-r2r} bash tools/round_measure_r2.sh
