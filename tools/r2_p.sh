set -u
o=gpurun_out/p; mkdir -p $o
for a in 32 64 256; do AGGLOM=$a timeout 900 python tools/dist_projection.py > $o/proj_$a.json 2> $o/proj_$a.err; done
python - <<'PY'
import json
for a in (32,64,256):
    try: p=json.loads(open(f'gpurun_out/p/proj_{a}.json').read().strip().splitlines()[-1])
    except Exception as e: print(a, 'fail', e); continue
    w=p['weak_config5']
    print(a, [(k, p[k]['kdist'], round(p[k]['projected_efficiency'],3)) for k in ('p2','p4','p8')], [(k, w[k]['kdist'], round(w[k]['projected_weak_efficiency'],3)) for k in ('p2','p4','p8')])
PY
