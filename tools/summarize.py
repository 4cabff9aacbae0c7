"""One-line summaries of bench JSON lines found in the given log files."""
import json
import sys

for f in sys.argv[1:]:
    for line in open(f):
        line = line.strip()
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        ph = {k.replace("us_", ""): round(v, 1) for k, v in (d.get("phases_us_median") or d.get("phases_us_diagnostic") or {}).items() if k != "note"}
        dn = d.get("dense_baseline") or {}
        print(f"{f}: {d['config']['workload']} N={d['n_gpus']} {d['value']/1e6:.1f} Mtok/s "
              f"{d.get('us_per_step', 0):.1f} us/step U_g={d.get('U_global')} phases={ph} "
              f"S4frac={d.get('roofline', {}).get('frac', 0):.3f} S56frac={((d.get('roofline_s5_s6') or {}).get('frac') or 0):.3f} "
              f"dense_us={1e3*dn.get('ms_per_step', 0):.1f} speedup={dn.get('speedup_unique_vs_dense', 0):.2f} "
              f"gate={dn.get('gate_0.8x', 0):.2f} e2e={((d.get('e2e') or {}).get('value') or 0)/1e6:.1f}M")
        for name, s in (d.get("supporting") or {}).items():
            print(f"    {name}: {s.get('us_per_step', 0):.1f} us/step U_g={s.get('U_global')} "
                  f"S4frac={s.get('S4_roofline_frac') or 0:.3f} S1={s.get('S1_us_diagnostic') or 0:.1f} "
                  f"dense_us={s.get('dense_us_per_step') or 0:.1f} "
                  f"speedup={s.get('speedup_unique_vs_dense') or 0:.2f} gate={s.get('gate_0.8x') or 0:.2f}")
