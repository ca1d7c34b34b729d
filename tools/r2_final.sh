#!/bin/bash
# Round-2 final measurement on one B200: smoke, the full GPU suite, every bench line
# (BASELINE configs + the 3-D lines, with CPU baselines), the reference arm, launch
# lists, ncu captures and the multi-GPU projection (tools/round_measure_r2.sh).
set -u
o=gpurun_out/${TAG:-final}
mkdir -p $o
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $o/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=30 > $o/gputest.log 2>&1
TAG=${TAG:-final} bash tools/round_measure_r2.sh
for c in 3d-poisson7-255 3d-aniso7-255 3d-checkeraniso7-255 3d-checker27-255 3d-poisson7-511; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 >> $o/configs3d.jsonl 2>> $o/configs3d.err
done
( time timeout 900 python bench.py --impl reference --steps 3 --warmup 3 ) > $o/reference.json 2> $o/reference.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
PROFILE=1 timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file $o/p7_launches.csv python tools/bench3.py poisson7 255 point > $o/ncu3d.log 2>&1
PROFILE=1 timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file $o/a7_launches.csv python tools/bench3.py aniso7 255 planes >> $o/ncu3d.log 2>&1
