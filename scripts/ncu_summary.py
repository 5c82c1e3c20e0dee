"""Text summary of one kernel in an ncu report (the profiles/*_ncu_details.txt format): every metric of the
details page, then selected raw metrics.  python scripts/ncu_summary.py REPORT.ncu-rep "header line" > out.txt"""
import csv
import io
import subprocess
import sys

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sass__inst_executed_local_loads",
       "sass__inst_executed_local_stores", "smsp__sass_inst_executed_op_shared_ld.sum",
       "smsp__sass_inst_executed_op_shared_st.sum", "lts__t_sectors_srcunit_tex_op_red.sum",
       "lts__t_requests_srcunit_tex_op_red.sum"]


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out[out.index('"'):] if '"' in out else out)))


def main():
    rep, header = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    print(header)
    print()
    rows = ncu_csv(rep, "details")
    hdr = rows[0]
    isec, imet, iunit, ival = (hdr.index(c) for c in ("Section Name", "Metric Name", "Metric Unit", "Metric Value"))
    for r in rows[1:]:
        if len(r) > ival:
            print(f"{r[isec]:40s} {r[imet]:52s} {r[ival]:>20s} {r[iunit]}")
    print()
    print("raw metrics:")
    raw = ncu_csv(rep, "raw")
    names, units, vals = raw[0], raw[1], raw[2]
    for m in RAW:
        if m in names:
            i = names.index(m)
            print(f"{m:70s} {vals[i]} {units[i]}")


if __name__ == "__main__":
    main()
