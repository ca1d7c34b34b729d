set -u
o=gpurun_out/z; mkdir -p $o
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $o/smoke.log 2>&1; tail -1 $o/smoke.log
timeout 1200 python -m pytest tests -q -m gpu > $o/gputest.txt 2>&1; tail -1 $o/gputest.txt
