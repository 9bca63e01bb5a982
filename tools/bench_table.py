"""Markdown table of a bench.py JSON line's per_config block (for DESIGN.md).

    python tools/bench_table.py profiles/r2m_bench.json
"""
import json
import sys

line = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
names = {"configs[0]": "configs[0] TTT B=1024", "configs[0]@2^22": "configs[0] TTT B=2²²",
         "configs[1]": "configs[1] C4 B=2²² (headline)", "configs[2]": "configs[2] Hex 11×11 B=2²²",
         "configs[3]": "configs[3] Reversi B=2²²", "configs[4]": "configs[4] Pente 19×19 B=2²²"}
print("| config | env steps/s | e2e (C-ABI host buffers) | e2e (Python API) | ALU-pipe roofline frac | "
      "CPU port (oracle, threads) | parity (envs checked / mismatches) |")
print("|---|---|---|---|---|---|---|")
for e in line["per_config"]:
    e2e = line["e2e"]["value"] if isinstance(e["e2e"], str) else e["e2e"]["value"]
    hc = e.get("e2e_python") if isinstance(e.get("e2e_python"), dict) else line.get("e2e_python")
    e2e_c = f"{hc['value'] / 1e9:.2f} G" if hc else "-"
    rl = e.get("roofline") or {}
    frac = rl.get("frac")
    cpu = e["cpu_baseline"]
    par = e["parity"]
    g = "G" if e["value"] >= 1e9 else "M"
    print(f"| {names.get(e['config'], e['config'])} | {e['value'] / 1e9:.2f} G | {e2e / 1e9:.2f} G | "
          f"{e2e_c} | "
          f"{'%.2f' % frac if frac else '-'} | {cpu['value'] / 1e6:.1f} M ({cpu['cores']}) | "
          f"{par['envs_checked']} / {par['mismatches']} |")
print()
print(f"headline {line['value'] / 1e9:.2f} G env steps/s, e2e {line['e2e']['value'] / 1e9:.2f} G, "
      f"clocks {line['clocks']}, roofline frac {line['roofline'].get('frac')}, "
      f"stale {line['roofline'].get('profile_stale')}")
env = line["env_step_api"]
print(f"env bool {env['env_steps_per_s'] / 1e9:.2f} G frac {env['roofline']['frac']:.3f}; "
      f"bits {env['bits_mask']['env_steps_per_s'] / 1e9:.2f} G frac {env['bits_mask']['roofline']['frac']:.3f}; "
      f"random step {line['step_kernel']['env_steps_per_s_upper'] / 1e9:.2f} G frac "
      f"{line['step_kernel']['roofline']['frac']:.3f}")
