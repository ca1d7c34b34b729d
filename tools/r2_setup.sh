set -u
o=gpurun_out/r2g; mkdir -p $o
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1
N=8191 WL=poisson timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $o/setup_launches.csv python tools/profile_setup.py > $o/ncu_setup.log 2>&1
N=4095 WL=aniso timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $o/setup_launches_aniso.csv python tools/profile_setup.py >> $o/ncu_setup.log 2>&1
N=8191 WL=poisson timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_rap_tiled -c 1 -o $o/rap_full python tools/profile_setup.py >> $o/ncu_setup.log 2>&1
