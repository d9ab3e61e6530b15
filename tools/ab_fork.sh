for c in C3 C4 C5; do for f in 1 0; do echo "$c fork=$f $(LFSR_ASM=1 LFSR_ASM_FORK=$f timeout 300 python tools/quick_time.py $c 10 2>&1 | tail -1 | python -c 'import json,sys
d=json.loads(sys.stdin.read()); print(round(d["it_per_s"],1), round(d["ms_per_iter"],4))')"; done; done
