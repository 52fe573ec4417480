"""BASELINE.md §5 / DESIGN.md §6 result rows from a bench line and the oracle's golden records
(dev tool): python tools/results_table.py profiles/r02_bench_C2.json"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d = json.load(open(sys.argv[1]))
peak = d["roofline"]["peak"]


def gold(cfg, prec, ortho, m):
    with open(os.path.join(ROOT, "tests", "golden", "full_size", f"{cfg}_{prec}_{ortho}_m{m}.json")) as f:
        return json.load(f)


def tts(ms):
    return f"{ms / 1e3:.2f} s" if ms >= 1000 else f"{ms:.1f} ms"


rows = []
configs = {"C2": (dict(d["variants"], m=50), 2097152, 14581760)}
for name, e in d["extra_configs"].items():
    configs[name] = (e, e["n"], e["nnz"])
print("| Config | P | ortho | precision | cycles (GPU / oracle) | inner (GPU / oracle) | TTS GPU | model GB/s (of 8 TB/s / of "
      f"{peak:.0f}) | TTS oracle (threads) | mixed/fp64 speedup |")
print("|---|---|---|---|---|---|---|---|---|---|")
for name, (e, n, nnz) in configs.items():
    for prec in ("mixed", "fp64"):
        for ortho in ("mgs", "cgsr"):
            v = e[f"{prec}_{ortho}"]
            g = gold(name, prec, ortho, e["m"])
            sp = f"{e[f'fp64_{ortho}']['tts_ms'] / v['tts_ms']:.2f}×" if prec == "mixed" else "–"
            gbps = v["model_GBps"]
            print(f"| {name} | 1 | {ortho.upper()} | {prec} | {v['cycles']} / {g['cycles']} | {v['inner_iters']} / {g['inner_iters']} | "
                  f"{tts(v['tts_ms'])} | {gbps:.0f} ({gbps / 8000:.2f} / {gbps / peak:.2f}) | "
                  f"{g['seconds']:.1f} s ({g['threads']}) | {sp} |")
print()
print("| config | variant | cycles / inner | TTS (ms) | SpMV / ortho (ms) | model GB/s | of peak |")
print("|---|---|---|---|---|---|---|")
for name, (e, n, nnz) in configs.items():
    for prec in ("mixed", "fp64"):
        for ortho in ("mgs", "cgsr"):
            v = e[f"{prec}_{ortho}"]
            ph = v.get("phase_ms") or {}
            print(f"| {name} | {prec} {ortho.upper()} | {v['cycles']} / {v['inner_iters']} | {v['tts_ms']:.1f} | "
                  f"{ph.get('spmv', float('nan')):.1f} / {ph.get('ortho', float('nan')):.1f} | {v['model_GBps']:.0f} | "
                  f"{v['model_GBps'] / peak:.2f} |")
r = d["roofline"]
print(f"\nbench: {d['value']:.1f} cycles/s, {d['ms_per_step']:.1f} ms/step, roofline {r['achieved']:.0f} GB/s = {r['frac']:.3f} of "
      f"{peak:.0f} ({r['frac_of_8TBps']:.3f} of 8 TB/s), e2e {d['e2e']['value']:.1f}; ilu0: "
      + json.dumps({k: (round(v["tts_ms"], 1) if isinstance(v, dict) and "tts_ms" in v else v) for k, v in d.get("ilu0_untimed", {}).items()})[:600])
