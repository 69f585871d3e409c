# SM clock / power while a config runs back to back (is the product phase power-capped?)
cfg=${1:-cfg2}; iters=${2:-3000}
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap,temperature.gpu --format=csv,noheader,nounits -lms 50 > gpurun_out/clk_$cfg.csv &
SMI=$!
sleep 0.5
python profiles/run_config.py $cfg --iters $iters
kill $SMI
python - <<PY
import statistics
rows=[l.strip().split(', ') for l in open('gpurun_out/clk_$cfg.csv') if l.strip()]
sm=[float(r[0]) for r in rows]; pw=[float(r[1]) for r in rows]
print('$cfg', 'samples', len(rows), 'sm_mhz median', statistics.median(sm), 'min', min(sm), 'max', max(sm), 'power max', max(pw), 'median', statistics.median(pw), 'capped', sum(1 for r in rows if r[2].strip()=='Active'))
PY
