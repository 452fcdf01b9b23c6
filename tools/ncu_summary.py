"""Summarise an ncu report: key metrics, stall reasons, SASS opcode mix per kernel."""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
def run(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout

raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
h, units = raw[0], raw[1]
keys = ['gpu__time_duration.sum', 'smsp__inst_executed.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum',
        'launch__registers_per_thread', 'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active', 'smsp__thread_inst_executed_per_inst_executed.ratio']
for r in raw[2:]:
    print("====", r[h.index("Kernel Name")][:70])
    for k in keys:
        if k in h:
            print(f"   {k:70s} {r[h.index(k)]} {units[h.index(k)]}")
    st = []
    for i, m in enumerate(h):
        if m.startswith('smsp__average_warps_issue_stalled_') and m.endswith('_per_issue_active.ratio'):
            try:
                v = float(r[i])
            except ValueError:
                continue
            st.append((v, m.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')))
    st.sort(reverse=True)
    print("   stalls:", ", ".join(f"{n}={v:.2f}" for v, n in st[:8]))
n = len(raw) - 2
for k in range(n):
    rows = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass",
                                           "--launch-skip", str(k), "--launch-count", "1"))))
    hh = rows[1]
    si, ie, sa = hh.index('Source'), hh.index('Instructions Executed'), hh.index('Warp Stall Sampling (All Samples)')
    ops, stl = collections.Counter(), collections.Counter()
    tot = tots = 0
    for r in rows[2:]:
        try:
            c, s = int(r[ie]), int(r[sa])
        except (ValueError, IndexError):
            continue
        t = r[si].strip().split()
        if not t:
            continue
        op = t[1] if t[0].startswith('@') else t[0]
        op = op.split('.')[0]
        ops[op] += c; stl[op] += s; tot += c; tots += s
    print("==== opcode mix", rows[0][1][:60], "warp-instrs", tot)
    print("   " + ", ".join(f"{o} {c / tot * 100:.1f}%/{stl[o] / max(1, tots) * 100:.0f}%st" for o, c in ops.most_common(16)))
