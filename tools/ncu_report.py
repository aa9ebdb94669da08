"""Text summary of an ncu --set full capture (for profiles/): SOL, pipes,
DRAM traffic per launch, stall reasons, top SASS hot spots."""
import csv, io, subprocess, sys
rep = sys.argv[1]
def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
IDX = int(sys.argv[2]) if len(sys.argv) > 2 else 0
h, v = raw[0], raw[2 + IDX]
d = dict(zip(h, v))
def g(k, default="?"):
    return d.get(k, default)
print(f"kernel: {g('Kernel Name')[:100]}")
units = dict(zip(h, raw[1]))
print(f"duration: {g('gpu__time_duration.sum')} {units.get('gpu__time_duration.sum', '')}  grid: {g('launch__grid_size')}  block: {g('launch__block_size')}  regs: {g('launch__registers_per_thread')}")
rd = float(g('dram__bytes_read.sum', 0) or 0); wr = float(g('dram__bytes_write.sum', 0) or 0)
unit = [u for k, u in zip(h, raw[1]) if k == 'dram__bytes_read.sum']
print(f"dram_bytes_read: {rd} {unit[0] if unit else ''}  dram_bytes_write: {wr}")
for k in h:
    if (('pipe_' in k and 'pct_of_peak_sustained_active' in k and '.avg.' in k) or
            k in ('sm__throughput.avg.pct_of_peak_sustained_elapsed', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
                  'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed',
                  'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
                  'lts__t_sector_hit_rate.pct', 'TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed')):
        try:
            if float(d[k]) > 0.5:
                print(f"  {k}: {d[k]}")
        except ValueError:
            pass
print("stall samples:")
st = sorted(((k, float(d[k])) for k in h if k.startswith('smsp__pcsamp_warps_issue_stalled') and 'not_issued' not in k
             and d[k] not in ('', None)), key=lambda x: -x[1])[:8]
for k, x in st:
    print(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}: {x:.0f}")
