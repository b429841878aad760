"""Top stall reasons + instruction mix per kernel from an ncu report (raw page)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[0]
for r in rows[2:]:
    name = r[hdr.index('Kernel Name')][:70]
    st = []
    for i, h in enumerate(hdr):
        if h.startswith('smsp__average_warps_issue_stalled_') and h.endswith('_per_issue_active.ratio'):
            try:
                st.append((float(r[i]), h[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]))
            except ValueError:
                pass
    st.sort(reverse=True)
    g = lambda k: r[hdr.index(k)] if k in hdr else "?"
    print("==", name, g('gpu__time_duration.sum'), "ms")
    print("   stalls:", ", ".join(f"{n}={v:.2f}" for v, n in st[:7]))
    print("   inst", g('smsp__inst_executed.sum'), "fp64 pipe %", g('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'),
          "ldg req", g('l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum'), "sectors", g('l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum'),
          "shared wavefronts", g('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum'), "dram rd", g('dram__bytes_read.sum'))
