mkdir -p gpurun_out
for i in 1 2; do for h in 1 0; do
LPASS_HOIST=$h timeout 300 python tools/latency_cfg1.py 200 > gpurun_out/lat_h$h.$i.json 2> gpurun_out/lat_h$h.$i.err; echo "hoist=$h run $i: $(grep -E 'fused_pass' gpurun_out/lat_h$h.$i.err | tr -s ' ' | cut -d' ' -f1-3 | tr '\n' ';')"
done; done
