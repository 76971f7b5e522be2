# A/B the working tree against the _ab_prev worktree (git worktree add _ab_prev <rev>)
# on the same box; extra env for the current side: CUR_ENV="VAR=1 ..."
B='import json,sys; l=json.loads(sys.stdin.read()); print(round(l["value"],1), round(l["e2e"]["value"],1), round(l["ms_per_step"],2))'
for i in 1 2; do
  echo -n "cur  "; env $CUR_ENV timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline | tail -1 | python -c "$B"
  echo -n "prev "; (cd _ab_prev && timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline | tail -1 | python -c "$B")
done
