# A/B of environment switches on bench cells: one process per (cell, variant), graph-replay time.
# usage: bash tools/ab_env.sh "<cells: wl:sel:q ...>" "<variants: NAME=V,NAME2=V2 | - ...>"
for cell in $1; do
  IFS=: read wl sel q <<< "$cell"
  n=""; [ "$wl" = c4 ] && n="--n 6250000"; [ "$wl" = c5 ] && n="--n 2500000"
  for v in $2; do
    envs=""; [ "$v" != "-" ] && envs=$(echo "$v" | tr ',' ' ')
    echo -n "[$v] "
    env $envs timeout 300 python tools/run_cell.py --workload $wl --sel $sel --q $q $n --reps 2 2>&1 | grep '^cell' | sed 's/ | .*//'
  done
done
