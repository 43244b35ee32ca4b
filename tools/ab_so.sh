for r in 1 2 3; do for v in ${SOS:-old new}; do cp abso/$v.so paper_2602_00879_b200/libdesmoe.so; timeout 300 python bench.py --no-cpu-baseline --strategies vote,vanilla --steps 100 --warmup 5 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['strategies']['vanilla']['us_per_block'], d['value_l2_flushed'])"; done; done
