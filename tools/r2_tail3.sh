set -u
o=gpurun_out/${TAG:-g3tail}; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu3d.py -q -x > $o/test.log 2>&1; tail -1 $o/test.log
b() { timeout 300 python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/x.json 2>> $o/err.log; python -c "import json; d=json.load(open('$o/x.json')); print('$1 $2', round(d['ms_per_step'],3), d['kernels_per_cycle'])"; }
b 3d-poisson7-255 tail
BMG3_NO_TAIL=1 b 3d-poisson7-255 notail
b 3d-checker27-255 tail
for t in 1024 4096 16384; do BMG3_PTAIL_MAX=$t b 3d-aniso7-255 ptail$t; done
