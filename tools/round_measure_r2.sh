#!/bin/bash
# Round-2 measurements in ONE gpurun call (run from the repo root):
# every BASELINE config through bench.py, the cycle launch lists (dram bytes) for the
# traffic rows, ncu --set full captures of the dominant kernels, setup launch lists,
# the multi-GPU projection.
set -u
out=gpurun_out/${TAG:-rm2}
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
run() { timeout 600 python bench.py "$@" >> $out/configs.jsonl 2>> $out/configs.err; }
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err
run --config poisson33 --steps 200 --no-cpu-baseline
run --config checker1025 --steps 100 --pcg 1 --no-cpu-baseline
run --config aniso4097 --steps 30 --e2e-steps 2 --no-cpu-baseline
run --config aniso4097 --relax yline --steps 30 --e2e-steps 2 --pcg 1 --no-cpu-baseline
run --config checker4096 --steps 50 --e2e-steps 2 --pcg 1 --no-cpu-baseline
run --config poisson8193 --steps 40 --no-cpu-baseline --e2e-steps 0 --nrhs 8
run --config poisson8193 --steps 40 --no-cpu-baseline --e2e-steps 0 --unfused
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
N=8191 WL=poisson NCYC=2 RELAX=0 timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file $out/cycle_launches.csv python tools/profile_cycle.py > $out/ncu.log 2>&1
N=1023 WL=checker NCYC=2 RELAX=0 timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file $out/cycle1023_launches.csv python tools/profile_cycle.py >> $out/ncu.log 2>&1
N=4095 WL=aniso NCYC=2 RELAX=0 timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file $out/cycle4095_launches.csv python tools/profile_cycle.py >> $out/ncu.log 2>&1
N=8191 WL=poisson NCYC=1 RELAX=0 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_fused" -c 3 -o $out/fused_full python tools/profile_cycle.py >> $out/ncu.log 2>&1
N=8191 WL=poisson timeout 300 ncu --metrics $M --clock-control none --csv --log-file $out/setup_launches.csv python tools/profile_setup.py >> $out/ncu.log 2>&1
N=4095 WL=aniso timeout 300 ncu --metrics $M --clock-control none --csv --log-file $out/setup_aniso_launches.csv python tools/profile_setup.py >> $out/ncu.log 2>&1
timeout 900 python tools/dist_projection.py > $out/dist_projection.json 2> $out/dist_projection.err
