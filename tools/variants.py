"""Build libbmg.so variants with -D tuning macros (kernels_fused.cu Inst) into tools/vlib/.

usage: python tools/variants.py NAME "-DBMG_E5DN=2 -DBMG_D5=3" [NAME FLAGS ...]
"""
import os, subprocess, sys
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__ as ge

out = os.path.join(ge.ROOT, "tools", "vlib")  # travels with gpurun (variants/ does not)
os.makedirs(out, exist_ok=True)
srcs = sorted(os.path.join(ge.CSRC, f) for f in os.listdir(ge.CSRC) if f.endswith(".cu"))


def build(name, flags):
    cmd = [ge._nvcc(), *ge.NVCC_FLAGS, *flags.split(), "-I", os.path.join(ge.ROOT, "include"), "-I",
           ge._nccl_include(), *srcs, "-o", os.path.join(out, f"libbmg_{name}.so"), "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return name, r.returncode, r.stderr[-400:]


args = sys.argv[1:]
with ThreadPoolExecutor(4) as ex:
    for name, rc, err in ex.map(lambda a: build(*a), zip(args[0::2], args[1::2])):
        print(name, "ok" if rc == 0 else "FAILED\n" + err)
