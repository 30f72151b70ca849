run() { (cd $1 && timeout 120 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items() if 'attn_bwd' in k})"); }
for i in 1 2; do run /root/repo; run /root/repo/ab_old2; done
