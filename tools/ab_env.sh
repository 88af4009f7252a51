# same-box comparison of env-selected kernel configurations (ENVS="A=1 B=2;C=3" ...)
IFS=';' read -ra CFGS <<< "$ENVS"
for rep in 1 2; do
  for cfg in "${CFGS[@]}"; do
    env $cfg timeout 300 python tools/kind_timing.py 2>&1 | grep -E "${KINDS:-grid}" | grep -v '"L": 16' | sed "s/^/[$cfg] /"
  done
done
