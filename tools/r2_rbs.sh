set -u
o=gpurun_out/${TAG:-g3s}; mkdir -p $o
compute-sanitizer --tool racecheck tools/mb_racecheck_bin > $o/mb_racecheck.txt 2>&1; tail -4 $o/mb_racecheck.txt
timeout 600 python -m pytest tests/test_gpu_fused_determinism.py -q -x > $o/det.log 2>&1; tail -2 $o/det.log
BMG3_RB=s timeout 900 python -m pytest tests/test_gpu3d.py -q -x > $o/test3d_s.log 2>&1; tail -2 $o/test3d_s.log
for v in s 16,32; do
  BMG3_RB=$v timeout 300 python bench.py --config 3d-poisson7-255 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/rb_$v.json 2>> $o/err.log
  python -c "import json,sys; d=json.load(open('$o/rb_$v.json')); print('$v', round(d['ms_per_step'],3), round(d['roofline']['sweep_ms'],4), round(d['roofline']['frac'],3))"
done
BMG3_RB=s timeout 600 ncu --set full --clock-control none -k regex:k3_rb7s -c 1 -o $o/rb7s_full python tools/bench3.py poisson7 255 point 1 > $o/ncu.log 2>&1
BMG3_RB=s timeout 300 compute-sanitizer --tool racecheck python tools/sanitize3d.py > $o/san3d_rc_s.txt 2>&1; tail -2 $o/san3d_rc_s.txt
