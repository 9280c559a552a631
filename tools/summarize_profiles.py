"""Summaries of a round's ncu captures for profiles/ (run here, no GPU needed).

    python tools/summarize_profiles.py r01

Reads gpurun_out/<round>_launches.csv (launch list of `python bench.py`),
gpurun_out/<round>_decode_full.ncu-rep and <round>_prefill_full.ncu-rep and
writes profiles/<round>_launches_summary.txt, profiles/<round>_decode_full.txt,
profiles/<round>_prefill_full.txt and profiles/decode_traffic.json.
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__shared_mem_per_block_dynamic",
]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        d["_units"] = dict(zip(hdr, units))
        res.append(d)
    return res


def c2_decode_bytes(layer):
    import paper_2406_14909_b200 as moa
    from moa_workloads import CONFIGS, rule_table
    cfg, t = CONFIGS["C2"], rule_table("C2")
    W = moa.resolve_spans(t["alpha"][layer], t["beta"][layer], cfg.N, cfg.n_sink)
    G = cfg.group
    wg = [max(W[g * G:(g + 1) * G]) for g in range(cfg.hkv)]
    d = cfg.head_dim
    rows = sum(cfg.n_sink + w for w in wg)
    return cfg.batch * (rows * d * 2 * 2 + cfg.hq * d * 2 * 2 + cfg.hkv * d * 2 * 2 * 2)


def main(rnd):
    out_dir = os.path.join(ROOT, "profiles")
    os.makedirs(out_dir, exist_ok=True)
    src = os.path.join(ROOT, "gpurun_out")
    # ---- launch list
    rows = list(csv.reader(open(os.path.join(src, f"{rnd}_launches.csv"))))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"])
    tot = sum(v[1] for v in agg.values())
    lines = [f"# {rnd}: ncu launch list of `python bench.py --steps 1 --warmup 3` (first launches of the timed",
             "# step after the warm-up; gpu__time_duration.sum, --clock-control none; cold-cache, serialised --",
             "# compare SHARES, not absolute times)",
             f"{'kernel':<40} {'launches':>8} {'total_us':>12} {'mean_us':>10} {'share':>7}"]
    for name, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{name:<40} {n:>8} {ns / 1e3:>12.1f} {ns / n / 1e3:>10.2f} {ns / tot:>7.1%}")
    with open(os.path.join(out_dir, f"{rnd}_launches_summary.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))
    # ---- full captures
    for kind in ("decode", "prefill"):
        rep = os.path.join(src, f"{rnd}_{kind}_full.ncu-rep")
        if not os.path.exists(rep):
            continue
        ms = raw_metrics(rep)
        with open(os.path.join(out_dir, f"{rnd}_{kind}_full.txt"), "w") as f:
            f.write(f"# {rnd}: ncu --set full --clock-control none, {kind} kernel "
                    f"(tools/prof_run.py, C2)\n")
            for m in ms:
                f.write(f"kernel: {m.get('Kernel Name', '')[:120]}\n")
                for k in KEYS:
                    f.write(f"  {k:<70} {m.get(k, 'n/a'):>16} {m['_units'].get(k, '')}\n")
        if kind == "decode":
            m = ms[0]
            unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd = float(m["dram__bytes_read.sum"]) * unit[m["_units"]["dram__bytes_read.sum"]]
            wr = float(m["dram__bytes_write.sum"]) * unit[m["_units"]["dram__bytes_write.sum"]]
            import re
            cross = re.search(r"decode_mma_kernel<\d+, \d+, \d+, (1|true)>", m.get("Kernel Name", "")) is not None
            alg = sum(c2_decode_bytes(l) for l in range(32)) if cross else c2_decode_bytes(12)
            with open(os.path.join(out_dir, "decode_traffic.json"), "w") as f:
                json.dump({"round": rnd, "bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                           "algorithmic_bytes_same_launch": alg, "traffic_over_algorithmic": (rd + wr) / alg,
                           "launch": ("cross-layer decode_mma_kernel, all 32 C2 layers, token N+1 (tools/prof_run.py "
                                      "layers), batch 8") if cross else
                                     "decode_mma_kernel, C2 layer 12 (tools/prof_run.py decode), batch 8",
                           "source": f"gpurun_out/{rnd}_decode_full.ncu-rep"}, f, indent=1)
            print("decode traffic", rd + wr, "algorithmic", alg, (rd + wr) / alg)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
