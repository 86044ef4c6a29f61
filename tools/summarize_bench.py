"""One-line summaries of bench.py JSON lines in log files (value, e2e, step and GEMM ms,
roofline fractions, per-kernel fractions, phase times, comm, planner).

    python tools/summarize_bench.py gpurun_out/r2_n4/*.log
"""
import json
import sys


def main():
    for path in sys.argv[1:]:
        for ln in open(path):
            if not ln.startswith("{"):
                continue
            d = json.loads(ln)
            print("==", path)
            if d.get("impl") == "reference":
                print("  reference", round(d["value"], 1), d["unit"], "cores", d["cpu_baseline"]["cores"])
                continue
            r = d["roofline"]
            print("  N=%d value %.4g e2e %.4g ms/step %.3f gemm %.3f frac %.3f burst %.3f sm %s %s" % (
                d["n_gpus"], d["value"], d["e2e"]["value"], d["ms_per_step"], r.get("gemm_ms_per_step") or 0,
                r["frac"] or 0, r.get("frac_burst") or 0, d["clocks"]["sm_mhz"], d["clocks"]["reasons"]))
            k = d.get("kernels") or {}
            print("  kernels", {n: round(v.get("hbm_frac", v.get("frac_burst", 0)), 3) for n, v in k.items()
                                if isinstance(v, dict)})
            print("  phases", {n: round(v, 4) for n, v in d["phase_ms"].items()})
            if "step_ms" in d:
                sp = d["step_ms"]
                print("  step ms min %.3f median %.3f max %.3f" % (sp["min"], sp["median"], sp["max"]))
            c = d.get("comm")
            if c:
                print("  comm a2a %.1f GB/s ag %.1f GB/s (ag %.3f ms for %.1f MB)" % (
                    c.get("a2a_bus_gbs") or 0, c.get("ag_bus_gbs") or 0, c.get("ag_ms") or 0,
                    (c.get("ag_bytes") or 0) / 1e6))
            p = d.get("planner")
            if p:
                print("  planner p=%s sed=%s inputs=%s" % (p["p"], p["sed"], {k_: v for k_, v in p["measured_inputs"].items()
                                                                           if k_ != "source"}))


if __name__ == "__main__":
    main()
