#!/bin/bash
# End-of-round measurement (after the tail-solve / RAP staging / 9-point changes):
# GPU tests, bench line, configs, reference arm, launch lists, ncu, multi-GPU projection.
set -u
out=gpurun_out/${TAG:-f2}
mkdir -p $out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $out/build_smoke.log 2>&1; tail -1 $out/build_smoke.log
timeout 1200 python -m pytest tests -q -m gpu --durations=5 > $out/gputest.txt 2>&1; tail -1 $out/gputest.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err; tail -c 300 $out/bench.json
run() { timeout 600 python bench.py "$@" >> $out/configs.jsonl 2>> $out/configs.err; }
run --config poisson33 --steps 200 --no-cpu-baseline
run --config checker1025 --steps 100 --pcg 1 --no-cpu-baseline
run --config aniso4097 --steps 30 --e2e-steps 2 --no-cpu-baseline
run --config aniso4097 --relax yline --steps 30 --e2e-steps 2 --pcg 1 --no-cpu-baseline
run --config checker4096 --steps 50 --e2e-steps 2 --pcg 1 --no-cpu-baseline
run --config poisson8193 --steps 40 --no-cpu-baseline --e2e-steps 0 --nrhs 8
run --config poisson8193 --steps 40 --no-cpu-baseline --e2e-steps 0 --unfused
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/reference.json 2> $out/reference.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
N=8191 WL=poisson NCYC=2 RELAX=0 timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file $out/cycle_launches.csv python tools/profile_cycle.py > $out/ncu.log 2>&1
timeout 1500 python tools/dist_projection.py > $out/dist_projection.json 2> $out/dist_projection.err
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
