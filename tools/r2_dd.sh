# tile / tail thresholds after the planner change (runtime env knobs, cycle only)
set -u
o=gpurun_out/dd; mkdir -p $o; rm -f $o/sweep.jsonl
for tp in 70000 0 20000 300000; do for tl in 1024 256 4096; do for w in checker:1023 poisson:8191 aniso:4095 poisson:2047; do
  r=$(BMG_TILE_POINTS=$tp BMG_TAIL_POINTS=$tl WL=${w%%:*} N=${w##*:} LEGS=cycle timeout 120 python tools/legbench.py 2>/dev/null | tail -1)
  echo "$tp $tl $r" >> $o/sweep.jsonl
done; done; done
cat $o/sweep.jsonl
