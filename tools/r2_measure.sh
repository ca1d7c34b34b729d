# One GPU call: build, full GPU tests, bench, cycle traffic + launch list, ncu of the 9-point down leg.
set -u
o=gpurun_out/${TAG:-r2c}
mkdir -p $o
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $o/build.log 2>&1
if [ "${TESTS:-1}" = 1 ]; then timeout 1500 python -m pytest tests -m gpu -q -x > $o/gputest.log 2>&1; fi
timeout 600 python bench.py --steps 20 --warmup 5 > $o/bench.json 2> $o/bench.err
N=8191 WL=poisson NCYC=2 RELAX=0 timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file $o/cycle_launches.csv python tools/profile_cycle.py > $o/ncu1.log 2>&1
if [ "${FULL9:-1}" = 1 ]; then
N=8191 WL=poisson NCYC=1 RELAX=0 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_fused_down -c 2 -o $o/fused_down_full python tools/profile_cycle.py > $o/ncu2.log 2>&1
fi
