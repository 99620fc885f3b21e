"""Summarise an ncu --set full report: key raw metrics + SASS opcode / stall histogram."""
import collections, csv, io, re, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__average_warp_latency_per_inst_issued.ratio",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum.per_second", "dram__bytes_write.sum.per_second"]
for w in want:
    if w in h:
        print(f"{w:90s} {v[h.index(w)]} {u[h.index(w)]}")
stalls = [(n, v[i]) for i, n in enumerate(h) if re.match(r"smsp__average_warps_issue_stalled_\w+_per_issue_active\.ratio", n)]
stalls = sorted(((n.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(x or 0)) for n, x in stalls), key=lambda t: -t[1])
print("stalls (warps per issue):", ", ".join(f"{n}={x:.2f}" for n, x in stalls[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
r2 = list(csv.reader(io.StringIO(src)))
hh = r2[1]; data = r2[2:]
ia, iss, isrc = hh.index("Instructions Executed"), hh.index("Warp Stall Sampling (All Samples)"), hh.index("Source")
ti = sum(int(r[ia] or 0) for r in data); ts = sum(int(r[iss] or 0) for r in data)
op, opi = collections.Counter(), collections.Counter()
for r in data:
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[isrc])
    o = m.group(2) if m else "?"
    op[o] += int(r[iss] or 0); opi[o] += int(r[ia] or 0)
print(f"SASS: {ti} warp-instructions, {ts} stall samples")
for o, c in opi.most_common(16):
    print(f"  {o:10s} instr {c:9d} ({c/ti:5.1%})  samples {op[o]/max(ts,1):5.1%}")
