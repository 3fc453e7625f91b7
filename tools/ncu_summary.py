"""Summarise an ncu report: key metrics, stall reasons, top source lines (SASS) by samples."""
import csv, subprocess, sys, collections, io
rep = sys.argv[1]
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
d = dict(zip(h, v)); un = dict(zip(h, u))
print(v[h.index('Kernel Name')][:100] if 'Kernel Name' in h else '')
for k in ['gpu__time_duration.sum', 'launch__registers_per_thread', 'launch__grid_size', 'sm__warps_active.avg.pct_of_peak_sustained_active',
          'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__thread_inst_executed_per_inst_executed.ratio',
          'sm__inst_executed.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct',
          'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum']:
    if k in d: print(f"  {k:60s} {d[k]} {un.get(k,'')}")
tot = float(d['smsp__pcsamp_sample_count'].replace(',', ''))
it = [(k, float(x.replace(',', ''))) for k, x in d.items() if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued') and x.replace(',', '').replace('.', '').isdigit()]
it.sort(key=lambda t: -t[1])
print("  stalls:", ", ".join(f"{k[33:]} {100*x/tot:.1f}%" for k, x in it[:8]))
src = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'], capture_output=True, text=True).stdout
if len(sys.argv) > 2:
    open(sys.argv[2], 'w').write(src)
