"""Scaling table from rank-by-rank emulations (tools/emulate_ranks.py JSON lines) plus the
single-GPU bench line: python tools/scaling_table.py profiles/r02n_*.json"""
import json
import sys

rows = []
for p in sys.argv[1:]:
    d = json.load(open(p))
    par = d.get("parity") or {}
    sd = par.get("S_D_noRP", {})
    worst = max([sd.get(k, {}).get("rel_l2_est_full", 0) for k in ("S", "D")] + [par.get("out_rel_l2_rp_sample", 0)])
    ms = [r["ms_per_apply"] for r in d["ranks"]]
    rows.append((d["cfg"], d["world"], d["ms_per_apply_max_over_ranks"], min(ms), d["points_per_s_emulated"],
                 d["exchange_bytes"]["est_ms_nvlink_900GBps"], worst if par else None))
rows.sort()
print("| config | ranks | ms / apply (max over ranks) | fastest rank | points/s (emulated) | exchange est. ms | parity vs reference |")
print("|---|---|---|---|---|---|---|")
for c, w, mx, mn, pps, ex, par in rows:
    print(f"| {c} | {w} | {mx:.1f} | {mn:.1f} | {pps / 1e6:.1f} M | {ex:.2f} | {par:.1e} |" if par is not None else
          f"| {c} | {w} | {mx:.1f} | {mn:.1f} | {pps / 1e6:.1f} M | {ex:.2f} | — |")
