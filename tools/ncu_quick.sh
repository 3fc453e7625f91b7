# quick counters of the transport kernel (C3, 2e6 photons)
python tools/prof_run.py c3 2e6 > gpurun_out/plain_q.log 2>&1 && \
ncu --clock-control none -k regex:transport_kernel -s 1 -c 1 --csv \
  --metrics gpu__time_duration.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__inst_executed.sum,smsp__pcsamp_warps_issue_stalled_no_instructions,smsp__average_warp_latency_issue_stalled_no_instruction.ratio,launch__registers_per_thread,smsp__pcsamp_warps_issue_stalled_long_scoreboard,smsp__pcsamp_warps_issue_stalled_wait,smsp__pcsamp_sample_count \
  python tools/prof_run.py c3 2e6 2>/dev/null | grep -v "^==" | python3 -c "
import csv,sys
for r in csv.reader(sys.stdin):
    if len(r)>14 and r[0]!='ID': print(r[12].ljust(70), r[13].ljust(10), r[14])
"
