import csv,sys,subprocess
rep=sys.argv[1]
out=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
hdr=rows[0]; units=rows[1]
want=['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed','sm__throughput.avg.pct_of_peak_sustained_elapsed','launch__registers_per_thread','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','lts__t_sectors_srcunit_tex_op_read.sum','l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum']
idx=[hdr.index(w) if w in hdr else None for w in want]
for r in rows[2:]:
  print({w.split('.')[0]:(r[i]+' '+units[i] if i is not None else None) for w,i in zip(want,idx)})
