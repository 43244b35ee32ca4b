# Front-kernel A/B on the GPU box: front timeline marks (tools/ffn_trace.py,
# L2 flushed) and the L2-flushed sweep for a few shapes, under env settings
# given as arguments ("" = default), e.g.
#   tools/ab_front.sh "" "DESMOE_FRONT_FLAGS=4"
CFGS=${CFGS:-c2 c3}
BLOCKS=${BLOCKS:-32,256}
i=0
for envs in "$@"; do
  i=$((i+1))
  for c in $CFGS; do
    for b in ${BLOCKS//,/ }; do
      env $envs python tools/ffn_trace.py --config $c --block $b --strategy vote --json gpurun_out/ab$i_$c_$b.json > /dev/null 2>&1
      python - "$envs" $c $b gpurun_out/ab$i_$c_$b.json <<'PY'
import json, sys
d = json.load(open(sys.argv[4]))
ks = ["front_logits", "front_activated", "front_selected", "front_v_gathered", "front_votes", "front_ranked", "front_coreset", "front_rerouted", "ffn_list_loaded"]
print(f"[{sys.argv[1] or 'default'}] {sys.argv[2]} N={sys.argv[3]}", " ".join(f"{k.replace('front_','')}={d[k][-1] if k!='ffn_list_loaded' else d[k][0]}" for k in ks if k in d), "span", d.get("kernel_span_us"), "combine_end", d.get("combine_end_us"))
PY
    done
  done
  env $envs python tools/sweep.py --configs ${CFGS// /,} --blocks $BLOCKS --steps 20 --no-cpu 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print('[$envs]', r['config'], r['block'], 'vote', r['vote']['us_per_block'], 'front', r['vote']['front_us'], 'vanilla', r['vanilla']['us_per_block'])
"
done
