"""Summarise an ncu report: key metrics, top stall reasons and hottest SASS lines."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
r = list(csv.reader(raw))
hdr = r[0]
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'smsp__inst_executed.sum', 'launch__grid_size', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'lts__t_sectors_srcunit_tex_op_write.sum', 'lts__t_sectors_srcunit_tex_op_read.sum']
for row in r[2:]:
    d = dict(zip(hdr, row))
    print('==', d['Kernel Name'][:60])
    for k in keys:
        print('   ', k, d.get(k), r[1][hdr.index(k)] if k in hdr else '')
    st = [(k, d[k]) for k in hdr if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio')]
    st = sorted(st, key=lambda x: -float(x[1] or 0))
    print('    stalls', [(k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''), round(float(v), 2)) for k, v in st[:8]])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(src))
if len(rows) > 2:
    h = rows[1]; body = rows[2:]
    isrc = h.index('Source'); iss = h.index('Warp Stall Sampling (All Samples)'); iex = h.index('Instructions Executed')
    def num(x):
        try: return int(x)
        except ValueError: return 0
    tot = sum(num(x[iss]) for x in body)
    print('samples', tot, 'inst', sum(num(x[iex]) for x in body))
    for i in sorted(sorted(range(len(body)), key=lambda i: -num(body[i][iss]))[:top]):
        print(f"{i:5d} {body[i][iss]:>6s} {body[i][iex]:>10s} {body[i][isrc][:90]}")
