set -u
o=gpurun_out/${TAG:-g3d}; mkdir -p $o
for m in 0 1; do compute-sanitizer --tool racecheck tools/mb_racecheck_bin $m > $o/mb_racecheck_$m.txt 2>&1; tail -2 $o/mb_racecheck_$m.txt; done
timeout 900 python -m pytest tests/test_gpu_fused_determinism.py -q -x > $o/det.log 2>&1; tail -2 $o/det.log
