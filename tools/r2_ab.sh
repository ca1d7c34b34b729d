set -u
o=gpurun_out/ab; mkdir -p $o
for rep in 1 2; do
for v in old new; do
  if [ $v = old ]; then export BMG_LIB=$PWD/tools/ablib/libbmg_old.so; else unset BMG_LIB; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $o/$v.json 2>$o/$v.err
  python -c "import json; d=json.load(open('$o/$v.json')); L=d['levels']['legs']; print('$v', round(d['ms_per_step'],4), round(L[0]['down_ms'],4), round(L[0]['up_ms'],4), round(L[1]['down_ms'],4), round(d['solve']['setup_device_ms'],2), d['clocks'])"
done
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
timeout 600 python -m pytest tests/test_gpu_dist.py -q -x -k bitwise > $o/loop.log 2>&1; tail -1 $o/loop.log
timeout 900 python -m pytest tests/test_gpu_dist_shim.py -q -x -k "multi_rank" > $o/shim.log 2>&1; tail -1 $o/shim.log
