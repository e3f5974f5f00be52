"""Write profiles/<TAG>_summary.md from a tools/gpu_round.sh run (gpurun_out/),
and copy the bench line and launch lists into profiles/ (the tracked record).

  python tools/round_summary.py r02b"""
import io
import json
import shutil
import sys
from contextlib import redirect_stdout
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))
import ncu_summary  # noqa: E402

tag = sys.argv[1]
G, P = ROOT / "gpurun_out", ROOT / "profiles"
bench = json.loads((G / f"bench_{tag}.json").read_text().strip().splitlines()[-1])
shutil.copy(G / f"bench_{tag}.json", P / f"{tag}_bench.json")
out = io.StringIO()
with redirect_stdout(out):
    b = bench
    ph = b["phase_ms"]
    print(f"# Round evidence `{tag}` (tools/gpu_round.sh on one B200)\n")
    print(f"Bench headline ({b['config']['workload']}): **{b['ms_per_step']:.2f} ms/step = "
          f"{b['value']:.3g} transitions/s** (enumerate {ph['enumerate']:.2f}, relax {ph['relax']:.2f} ms); "
          f"e2e through dp_plan() {b['e2e']['value']:.3g}/s; parity {b['parity']}; "
          f"clocks {b['clocks']}; CPU port {b['cpu_baseline']['value']:.3g}/s on "
          f"{b['cpu_baseline']['cores']} threads; Python reference "
          f"{(b['cpu_baseline'].get('python_reference') or {}).get('value', float('nan')):.3g}/s on 1 core.\n")
    r = b["roofline"]
    print(f"Roofline (binding pipe): {r['bound']}: achieved {r['achieved']:.4g} of {r['peak']:.4g} "
          f"{r['unit']} = frac {r['frac']:.3f} (floor {r['floor_ms']:.2f} ms vs relax {r['relax_ms']:.2f} ms); "
          f"HBM byte model frac {r['hbm']['frac']:.2f}; measured DRAM per heavy launch: see captures.\n")
    print("## Configs (same run)\n\n| config | device ms | e2e ms | parity |\n|---|---|---|---|")
    for c in b["configs"]:
        dm = c.get("device_ms")
        print(f"| {c['config']} | {'' if dm is None else f'{dm:.2f}'} | {c.get('e2e_ms', float('nan')):.2f} | "
              f"{c.get('parity', c.get('error'))} |")
    for name, what in (("unet8", "U-Net c=8 (headline)"), ("c5p02", "C5 random-dag n=516 p=0.2 (north-star graph)")):
        lf = G / f"launches_{name}_{tag}.csv"
        if lf.exists():
            shutil.copy(lf, P / f"{tag}_{name}_launches.csv")
            print(f"\n## Launch list, {what} (one solve, ncu gpu__time_duration, cold-cache serialised)\n")
            ncu_summary.launches(str(lf))
        rep = G / f"prof_{name}_{tag}.ncu-rep"
        if rep.exists():
            print(f"\n## ncu --set full, heaviest relaxation launch of {what}\n")
            ncu_summary.capture(str(rep))
            print()
            ncu_summary.stalls(str(rep))
(P / f"{tag}_summary.md").write_text(out.getvalue())
print(out.getvalue()[:3000])
