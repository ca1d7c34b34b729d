set -u
o=gpurun_out/${TAG:-g3w}; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu3d.py -q -x > $o/test.log 2>&1; tail -1 $o/test.log
for c in 3d-aniso7-255 3d-poisson7-255; do
timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/x.json 2>> $o/err.log; python -c "import json; d=json.load(open('$o/x.json')); print('$c', round(d['ms_per_step'],3), d['kernels_per_cycle'], round(d['roofline']['sweep_ms'],3), round(d['roofline']['frac'],3))"
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
PROFILE=1 timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file $o/a7_launches.csv python tools/bench3.py aniso7 255 planes > $o/ncu.log 2>&1
python tools/launches.py $o/a7_launches.csv 100000 1 2>/dev/null | head -12
