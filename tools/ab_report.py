import glob, json, sys
for f in sorted(glob.glob("gpurun_out/abe_*.log")):
    lines = open(f).read().splitlines()
    js = [l for l in lines if l.startswith("{")]
    if not js:
        print(f, "FAILED", lines[-3:]); continue
    d = json.loads(js[-1]); k = d["kernel_ms"]
    print(f"{lines[-1]:40s} {d['value']:7.3f} s  gemm {k['gemm']:7.0f} fwd {k['solve_fwd']:6.0f} bwd {k['solve_bwd']:6.0f} ea {k['extend_add']:5.0f} trsm {k['trsm']:5.0f} diag {k['diag']:5.0f}")
    if len(sys.argv) > 1:
        print("   fwd", d["solve_ms_by_level"]["solve_fwd_by_level"]); print("   bwd", d["solve_ms_by_level"]["solve_bwd_by_level"])
