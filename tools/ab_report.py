"""Summarise tools/gpu_ab_env.sh bench logs (gpurun_out/abe_*.log)."""
import glob
import json
import sys

for f in sorted(glob.glob("gpurun_out/abe_*.log")):
    lines = open(f).read().splitlines()
    js = [l for l in lines if l.startswith("{")]
    if not js:
        print(f, "FAILED", lines[-3:])
        continue
    d = json.loads(js[-1])
    k = d["kernel_ms"]
    print(f"{lines[-1]:40s} {d['value']:7.3f} s  gemm {k['gemm']:6.0f} fwd {k['solve_fwd']:5.0f} bwd {k['solve_bwd']:5.0f} "
          f"green {k.get('green', 0):4.0f} ea {k['extend_add']:4.0f} trsm {k['trsm']:4.0f} diag {k['diag']:4.0f} elem {k['elem']:4.0f}")
    if len(sys.argv) > 1:
        for key, v in d["solve_ms_by_level"].items():
            print("   ", key, [round(x) for x in v])
