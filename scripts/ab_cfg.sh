# usage: bash scripts/ab_cfg.sh "<configs>" [bench args] -- A/B every alt lib on the given configs
cfgs=$1; shift
for c in $cfgs; do
  echo "### cfg$c"
  bash scripts/ab.sh --config $c "$@"
done
