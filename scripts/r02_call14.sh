tag=${1:-r02m}
bash scripts/r02_evidence.sh ${tag}
