"""Summarise ncu captures (launch list + full-set reports) into profiles/."""
import csv, collections, io, json, subprocess, sys

def launches(path, only_ours=True):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); ui = h.index('Metric Unit')
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi: continue
        v = float(r[vi].replace(',', ''))
        u = r[ui]
        v = v / 1e6 if u in ('nsecond', 'ns') else v / 1e3 if u in ('usecond', 'us') else v
        name = r[ki].split('(')[0].replace('void ', '').replace('eigb::<unnamed>::', '')
        if only_ours and 'eigb' not in r[ki] and 'unnamed>::' not in r[ki]:
            continue
        a = agg.setdefault(name, [0.0, 0]); a[0] += v; a[1] += 1
    return agg

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem']

def full(rep):
    """One entry per captured kernel launch of the report."""
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {'kernel': v[h.index('Kernel Name')][:80]}
        for k in KEYS:
            if k in h:
                d[k] = v[h.index(k)] + (' ' + units[h.index(k)] if units[h.index(k)] else '')
        res.append(d)
    return res

if __name__ == '__main__':
    res = {}
    if sys.argv[1].endswith('.csv'):
        agg = launches(sys.argv[1]); tot = sum(a[0] for a in agg.values())
        res = {k: {'ms': round(v, 4), 'launches': c, 'share': round(v / tot, 4)} for k, (v, c) in
               sorted(agg.items(), key=lambda x: -x[1][0])}
    else:
        for rep in sys.argv[1:]:
            res[rep] = full(rep)
    print(json.dumps(res, indent=1))
