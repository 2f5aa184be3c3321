#!/bin/bash
# A/B of the Hashing / OSNAP kernel shape (c4, OSNAP s = 4)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for flags in "" "-DFD_HASH_COLS=32 -DFD_HASH_CTAS=6" "-DFD_HASH_COLS=32 -DFD_HASH_CTAS=3" "-DFD_HASH_CTAS=2"; do
  FD_NVCC_EXTRA="$flags" python build.py > /dev/null 2>&1
  echo "=== [$flags]"
  timeout 300 python -m pytest tests -q -m gpu -k hash_parity_c2 2>&1 | tail -1
  timeout 600 python bench.py --variant osnap --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['ms_per_step'])"
done
python build.py > /dev/null 2>&1
