mkdir -p gpurun_out
timeout 900 python tools/depth_sweep.py --llama3-8b --seq 8192 --stream > gpurun_out/g32_s8192_stream.json 2> gpurun_out/g32_a.err; echo "a rc=$?"
timeout 900 python tools/depth_sweep.py --llama3-8b --seq 8192 --stream --cascade > gpurun_out/g32_s8192_stream_cascade.json 2> gpurun_out/g32_b.err; echo "b rc=$?"
timeout 900 python tools/depth_sweep.py --llama3-8b --seq 4096 > gpurun_out/g32_s4096.json 2> gpurun_out/g32_c.err; echo "c rc=$?"
timeout 600 python tools/depth_sweep.py > gpurun_out/g32_small.json 2> gpurun_out/g32_d.err; echo "d rc=$?"
for f in gpurun_out/g32_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', {k: d[k] for k in d if k in ('spearman','fit_c_over_eps','fit_log_rms_residual','estimate_seconds','peak_hbm_gb','mode')}, [round(x,2) for x in d.get('per_layer_paramgrad_response_over_eps',[])[:3]], '...', [round(x,2) for x in d.get('per_layer_paramgrad_response_over_eps',[])[-2:]])"; done
