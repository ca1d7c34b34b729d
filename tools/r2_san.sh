set -u
o=gpurun_out/san2; mkdir -p $o
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize3d.py > $o/san3d_$t.txt 2>&1
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_tile.py > $o/santile_$t.txt 2>&1
  timeout 1200 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_fused.py > $o/sanfused_$t.txt 2>&1
done
for f in $o/*.txt; do echo "== $f"; tail -3 $f; done
