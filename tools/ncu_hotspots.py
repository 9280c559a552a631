"""Read an ncu report (--set full --import-source on) here and print the kernel's headline
metrics, its SASS opcode mix and the instructions with the most warp-stall samples.

    python tools/ncu_hotspots.py gpurun_out/<name>.ncu-rep [--top 30]
"""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict

STALLS = ['stall_barrier', 'stall_branch_resolving', 'stall_dispatch', 'stall_drain', 'stall_lg', 'stall_long_sb',
          'stall_math', 'stall_membar', 'stall_mio', 'stall_misc', 'stall_no_inst', 'stall_not_selected',
          'stall_selected', 'stall_short_sb', 'stall_sleep', 'stall_tex', 'stall_wait']
HEAD = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread"]


def main(rep, top=30):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(d.get("Kernel Name", "")[:100])
        for k in HEAD:
            print(f"  {k:70s} {d.get(k, 'n/a')}")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hdr = rows[1]
    ia, isrc = hdr.index("Instructions Executed"), hdr.index("Source")
    idx = [hdr.index(k) for k in STALLS]
    ops, ops_st, tot_st = Counter(), Counter(), Counter()
    lines = []
    for i, r in enumerate(rows[2:]):
        if len(r) <= ia:
            continue
        n = int(r[ia] or 0)
        s = r[isrc].strip()
        op = s.split()[0] if s else "?"
        if op.startswith("@"):
            op = s.split()[1]
        op = op.split(".")[0]
        st = {k: int(r[j] or 0) for k, j in zip(STALLS, idx)}
        ops[op] += n
        ops_st[op] += sum(st.values())
        for k, v in st.items():
            tot_st[k] += v
        lines.append((sum(st.values()), i, n, s[:80], {k: v for k, v in st.items() if v}))
    tot = sum(ops.values())
    ts = sum(ops_st.values()) or 1
    print(f"\ninstructions executed {tot}, stall samples {ts}")
    for op, n in ops.most_common(25):
        print(f"  {op:12s} {n:12d} {n / tot * 100:5.1f}%   samples {ops_st[op] / ts * 100:5.1f}%")
    print("\nstall reasons (all samples):")
    for k, v in tot_st.most_common(12):
        print(f"  {k:24s} {v / ts * 100:5.1f}%")
    print(f"\ntop {top} instructions by stall samples:")
    lines.sort(reverse=True)
    for smp, i, n, s, st in lines[:top]:
        top3 = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        print(f"  #{i:5d} n={n:9d} smp={smp:6d} {s:60s} {top3}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30)
