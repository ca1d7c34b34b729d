set -u
o=gpurun_out/${TAG:-g3q}; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu3d.py -q -x > $o/test.log 2>&1; tail -3 $o/test.log
for a in "3d-poisson7-255" "3d-aniso7-255" "3d-checker27-255"; do
  timeout 300 python bench.py --config $a --steps 10 --warmup 3 --no-cpu-baseline >> $o/bench3.jsonl 2>> $o/bench3.err
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
PROFILE=1 timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file $o/p7_launches.csv python tools/bench3.py poisson7 255 point > $o/ncu.log 2>&1
PROFILE=1 timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file $o/c27_launches.csv python tools/bench3.py checker27 255 point >> $o/ncu.log 2>&1
