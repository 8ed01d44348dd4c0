# host-overhead variance experiment: bench with and without the NVML sampler, then a long trace
for i in 1 2 3; do python bench.py --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('sampler', round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['api_wall_ms_per_step'].items()})"; done
for i in 1 2 3; do MLK_BENCH_NO_SAMPLER=1 python bench.py --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('nosampler', round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['api_wall_ms_per_step'].items()})"; done
MLK_TRACE=1 python bench.py --no-cpu-baseline --steps 20 --e2e-steps 0 > gpurun_out/trace_hv.log 2>&1
