"""Summarise an ncu capture and a launch list into profiles/ (run in the build
container after a gpurun call brought the reports back).

    python tools/summarize_profile.py ROUND TAG report.ncu-rep launches.csv bench.json
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "launch__grid_size", "launch__block_size", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    res = []
    for r in rows[2:]:
        d = dict(zip(rows[0], r))
        res.append({"kernel": d.get("Kernel Name", "")[:120],
                    **{k: (d.get(k), rows[1][rows[0].index(k)] if k in rows[0] else None)
                       for k in KEYS}})
    return res


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    agg = {}
    for r in rows:
        name = r[4].split("(")[0]
        v = float(r[-1].replace(",", ""))
        if v != v:  # a launch ncu could not time (e.g. cut off at exit)
            continue
        agg.setdefault(name, [0, 0.0])
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    return [{"kernel": k, "launches": v[0], "ns": v[1], "share": v[1] / tot}
            for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])]


def main():
    rnd, tag, rep, lau, bench = sys.argv[1:6]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    prefix = os.path.join(ROOT, "profiles", f"r{int(rnd):02d}_{tag}")
    full = raw(rep)
    json.dump(full, open(prefix + "_ncu_full.json", "w"), indent=1)
    ll = launches(lau)
    json.dump(ll, open(prefix + "_launches.json", "w"), indent=1)
    subprocess.run(["cp", lau, prefix + "_launches.csv"])
    b = json.load(open(bench))
    json.dump(b, open(prefix + "_bench.json", "w"), indent=1)
    with open(prefix + "_summary.md", "w") as f:
        f.write(f"# round {rnd} — {tag}\n\n")
        f.write(f"bench: {b['value']:.1f} {b['unit']} ({b['ms_per_step']:.3f} ms/step, mode "
                f"{b.get('mode', b['config'].get('mode'))}), clocks {b['clocks']}\n\n")
        f.write("## launch list (ncu gpu__time_duration.sum, cold-cache, serialised)\n\n")
        f.write("| kernel | launches | total us | share |\n|---|---|---|---|\n")
        for r in ll:
            f.write(f"| {r['kernel'][:70]} | {r['launches']} | {r['ns'] / 1e3:.1f} | {r['share']:.1%} |\n")
        f.write("\n## full capture of the top kernel\n\n")
        for k in full:
            f.write(f"### {k['kernel']}\n\n")
            for key in KEYS:
                v, u = k[key]
                f.write(f"- {key}: {v} {u or ''}\n")
            f.write("\n")
    print("wrote", prefix + "_*")


if __name__ == "__main__":
    main()
