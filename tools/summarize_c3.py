"""Summarise full ncu captures of the config-3 kernels into profiles/.

    python tools/summarize_c3.py ROUND bench.json name=report.ncu-rep ...
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from summarize_profile import KEYS, ROOT, raw  # noqa: E402


def main():
    rnd, bench = sys.argv[1:3]
    b = json.load(open(bench))
    c3 = b.get("c3", {})
    prefix = os.path.join(ROOT, "profiles", f"r{int(rnd):02d}_c3")
    out = {}
    with open(prefix + "_summary.md", "w") as f:
        f.write(f"# round {rnd} — config-3 kernels (ncu --set full --clock-control none, one launch each, batch 1024)\n\n")
        for dt, v in c3.items():
            f.write(f"- bench {dt}: fast update {v['fast_ms']:.3f} ms ({v['fast_roofline']['frac']:.1%} of "
                    f"the FMA pipe), FWHT {v['fwht_ms']:.3f} ms ({v['fwht_roofline']['frac']:.1%} of HBM)\n")
        f.write("\n")
        for arg in sys.argv[3:]:
            name, rep = arg.split("=", 1)
            rows = raw(rep)
            out[name] = rows
            for k in rows:
                f.write(f"## {name}: {k['kernel']}\n\n")
                for key in KEYS:
                    val, unit = k[key]
                    f.write(f"- {key}: {val} {unit or ''}\n")
                f.write("\n")
    json.dump(out, open(prefix + "_ncu_full.json", "w"), indent=1)
    print("wrote", prefix + "_summary.md")


if __name__ == "__main__":
    main()
