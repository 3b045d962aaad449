for f in "$@"; do echo "== $f"; ncu -i $f --page details --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin))
want=['Duration','DRAM Throughput','Issue Slots Busy','L2 Hit Rate','Mem Busy','Executed Instructions','Dynamic Shared Memory Per Block','Achieved Occupancy','Warp Cycles Per Issued Instruction']
print('  '+'; '.join(x[12]+'='+x[14] for x in r[1:] if x[12] in want))
"; ncu -i $f --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
out=[]
for k,x in zip(h,v):
  if 'smsp__pcsamp_warps_issue_stalled' in k and not k.endswith('not_issued') :
    try:
      if float(x)>0: out.append((int(float(x)),k.replace('smsp__pcsamp_warps_issue_stalled_','')))
    except: pass
print('  stalls', sorted(out,reverse=True)[:7])
d={k:x for k,x in zip(h,v)}
print('  dram MB r/w', d.get('dram__bytes_read.sum'), d.get('dram__bytes_write.sum'), 'smem conflicts', d.get('l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum'))
"; done
