"""Print the key fields of bench JSON lines (gpurun_out/lines/<cfg>.log)."""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as exc:  # noqa: BLE001
        print(path, "no JSON line:", exc)
        continue
    print("==", path, d["config"]["workload"][:70])
    print("  ms", round(d["ms_per_step"], 3), "tok/s", round(d["value"]),
          "e2e", d.get("e2e") and round(d["e2e"]["ms_per_step"], 3))
    if d.get("roofline"):
        print("  roofline", {k: d["roofline"][k] for k in ("achieved", "peak", "frac", "peak_kind")})
    print("  dense", d.get("dense_ms"), "speedup", d.get("speedup_vs_fastest_dense"))
    print("  parity", {k: v for k, v in (d.get("parity") or {}).items() if k != "heads"})
    print("  cpu", d.get("cpu_baseline"))
    print("  clocks", d.get("clocks"), "launches", d.get("gpu_launches"), "cold", d.get("cold_step_ms"))
    if d.get("stack"):
        s = dict(d["stack"])
        s.pop("layer_ms_last_step", None)
        print("  stack", s)
    print("  key clusters", d.get("key_clusters_rank0"))
