"""One-line summary of bench.py JSON output files (for gpurun logs)."""
import json
import sys

for path in sys.argv[1:]:
    try:
        with open(path) as f:
            d = json.loads([l for l in f if l.startswith("{")][-1])
    except Exception as e:  # noqa: BLE001
        print(path, "unreadable:", e)
        continue
    r = d.get("roofline") or {}
    st = {k: round(v * 1000, 1) for k, v in (r.get("stage_ms_per_step") or {}).items()}
    lz = d.get("lanczos")
    print(f"{path}: {d.get('config', {}).get('workload')} value={d['value']:.1f} ms/step={d['ms_per_step']:.4f} "
          f"e2e={(d.get('e2e') or {}).get('value', 0):.1f} launches={d.get('gpu_launches')} "
          f"roof={r.get('bound')}:{r.get('frac', 0):.3f}({r.get('kernel')}) stages_us={st}"
          + (f" lanczos it={lz['iterations']} solve={lz['solve_s']:.3f}s" if lz else ""))
