"""Summarise an .ncu-rep: key throughput metrics + top stall reasons (run here, no GPU needed).
  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--json]"""
import csv, io, json, subprocess, sys

KEYS = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size', 'launch__shared_mem_per_block_dynamic',
        'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'lts__t_sector_hit_rate.pct', 'lts__t_bytes.sum', 'sm__cycles_elapsed.avg.per_second']


def raw(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def main():
    path = sys.argv[1]
    res = []
    for d, u in raw(path):
        e = {k: d[k] for k in KEYS if k in d}
        st = {k[len('smsp__pcsamp_warps_issue_stalled_'):]: float(v) for k, v in d.items()
              if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued')
              and v.replace('.', '', 1).isdigit()}
        tot = sum(st.values()) or 1
        e['stalls_pct'] = {k: round(v / tot * 100, 1) for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]}
        e['units'] = {k: u.get(k, '') for k in KEYS if k in d}
        res.append(e)
    if '--json' in sys.argv:
        print(json.dumps(res, indent=1))
    else:
        for e in res:
            for k, v in e.items():
                if k != 'units':
                    print(f'{k:60s} {v} {e["units"].get(k, "") if isinstance(v, str) else ""}')
            print()


if __name__ == '__main__':
    main()
