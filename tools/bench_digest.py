"""Print the headline fields of bench.py JSON lines (files given on the command line)."""
import json
import sys

for path in sys.argv[1:]:
    try:
        line = [l for l in open(path) if l.startswith("{")][-1]
        j = json.loads(line)
    except Exception as e:  # noqa: BLE001
        print(path, "unreadable:", e)
        continue
    r, c = j.get("roofline") or {}, j.get("config") or {}
    e2e, cpu, clk = j.get("e2e") or {}, j.get("cpu_baseline") or {}, j.get("clocks") or {}
    op = (r.get("operator_phases_only") or {}).get("frac")
    print(f"{path}: {c.get('workload')} engine {c.get('engine')} value {j.get('value'):.5g} {j.get('unit')} "
          f"ms/step {j.get('ms_per_step'):.1f} frac {r.get('frac')} (op-only {op}) achieved {r.get('achieved')} "
          f"peak {r.get('peak')} traffic {r.get('traffic')} e2e {e2e.get('value')} cpu {cpu.get('value')} "
          f"clocks {clk.get('sm_mhz')} {clk.get('reasons')} launches {j.get('gpu_launches')} "
          f"cg_steps {c.get('cg_steps_per_em_iter')} padded {c.get('probe_tile_cols_multiplied_over_active')}")
