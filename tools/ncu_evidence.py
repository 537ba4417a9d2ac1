"""Evidence summary of one ncu --set full capture for profiles/: duration, DRAM
bytes, L2 hit rate, L2 RED traffic, shared-memory pipe, instructions, stalls and
the hottest source lines.    python tools/ncu_evidence.py <rep> [records]"""
import csv, subprocess, sys
rep = sys.argv[1]
recs = float(sys.argv[2]) if len(sys.argv) > 2 else 100e6
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines())); h, u, v = r[0], r[1], r[2]
def g(k):
    return (v[h.index(k)] + ' ' + u[h.index(k)]).strip() if k in h else 'n/a'
print('kernel            ', g('Kernel Name'))
print('grid x block      ', g('launch__grid_size'), 'x', g('launch__block_size'), ' regs/thread', g('launch__registers_per_thread'),
      ' dyn smem', g('launch__shared_mem_per_block_dynamic'))
print('duration          ', g('gpu__time_duration.sum'))
print('DRAM read / write ', g('dram__bytes_read.sum'), '/', g('dram__bytes_write.sum'))
print('L2 sector hit rate', g('lts__t_sector_hit_rate.pct'))
print('L2 RED requests   ', g('lts__t_requests_op_red.sum'), ' sectors', g('lts__t_sectors_op_red.sum'),
      ' (global REDs issued:', g('l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum') + ')')
print('warp instructions ', g('smsp__inst_executed.sum'), ' = %.0f thread-instr/record' % (float(v[h.index('smsp__inst_executed.sum')].replace(',', '')) * 32 / recs),
      ' IPC', g('sm__inst_executed.avg.per_cycle_active'))
print('LSU data pipe     ', g('l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed'), '% of peak;  shared ld/st/atom wavefronts',
      g('l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum'), '/', g('l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum'), '/',
      g('l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum'))
print('shared bank conflicts (ld/st/atom)', g('l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum'), '/',
      g('l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum'), '/', g('l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum'))
print('shared atomic instr', g('smsp__inst_executed_op_shared_atom.sum'), ' red', g('smsp__inst_executed_op_shared_red.sum'))
tot = 0; out = []
for i, k in enumerate(h):
    if k.startswith('smsp__pcsamp_warps_issue_stalled_') and not k.endswith('_not_issued'):
        try:
            x = float(v[i].replace(',', '')); out.append((x, k[33:])); tot += x
        except ValueError:
            pass
print('stalls            ', ' '.join(f'{k}:{100*x/tot:.1f}%' for x, k in sorted(out, reverse=True)[:9]))
src = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source=cuda,sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines())); f = None; agg = []
for x in rows:
    if x and x[0] == 'File Path':
        f = x[1].split('/')[-1]; continue
    if len(x) >= 10 and x[0] and x[0] != 'Line No' and x[2] == '-':
        try:
            agg.append((int(x[4]), int(x[7]), f, x[0], x[1][:96]))
        except ValueError:
            pass
ts = sum(a[0] for a in agg); ti = sum(a[1] for a in agg)
print('hottest source lines (stall samples %, instructions %):')
for a in sorted(agg, key=lambda x: -x[0])[:18]:
    print(f'  {a[0]*100/ts:5.1f}%st {a[1]*100/ti:5.1f}%in {a[2]}:{a[3]} {a[4]}')
