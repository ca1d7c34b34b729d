set -u
o=gpurun_out/${TAG:-gblk}; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_parity.py -q -x > $o/test.log 2>&1; tail -2 $o/test.log
timeout 600 python bench.py --config poisson8193 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --nrhs 8 > $o/b8.json 2> $o/b8.err
python -c "import json; d=json.load(open('$o/b8.json')); print(d['ms_per_step'], json.dumps(d.get('block'))[:600])"
timeout 600 python bench.py --config checker4096 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --nrhs 4 > $o/b4.json 2>> $o/b8.err
python -c "import json; d=json.load(open('$o/b4.json')); print(d['ms_per_step'], json.dumps(d.get('block'))[:600])"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
N=8191 WL=poisson NRHS=8 NCYC=1 timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file $o/block8_launches.csv python tools/profile_cycle.py > $o/ncu.log 2>&1
