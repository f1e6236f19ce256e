"""Summarise an ncu --set full report (raw page) into the key roofline / pipe / stall metrics."""
import csv
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'sm__cycles_elapsed.avg.per_second', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_bytes.sum',
        'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'sm__memory_throughput.avg.pct_of_peak_sustained_elapsed']
STALL = 'smsp__average_warps_issue_stalled_'


def raw(path):
    """One dict per captured kernel launch: metric -> (unit, value)."""
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return [{h: (u, v) for h, u, v in zip(rows[0], rows[1], r)} for r in rows[2:]]


def summary(path):
    res = []
    for r in raw(path):
        d = {'kernel': r.get('Kernel Name', ('', ''))[1][:80]}
        d.update({k: f"{r[k][1]} {r[k][0]}".strip() for k in KEYS if k in r})
        st = {k[len(STALL):].replace('_per_issue_active.ratio', ''): float(v[1]) for k, v in r.items()
              if k.startswith(STALL) and k.endswith('_per_issue_active.ratio') and v[1]}
        d['stalls'] = {k: round(v, 3) for k, v in sorted(st.items(), key=lambda x: -x[1]) if v > 0.02}
        res.append(d)
    return res


if __name__ == '__main__':
    import json
    for p in sys.argv[1:]:
        print(p)
        print(json.dumps(summary(p), indent=1))
