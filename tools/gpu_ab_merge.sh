cd "${GRAFT_REPO_ROOT:-.}"
for rep in 1 2; do
for m in ${MERGES:-750,250 1500,250 2000,250 1500,150 1500,350 2000,350 1200,300}; do
  TT_DAG_MERGE=$m timeout -s KILL 120 python tools/dag_bandsweep.py lu 2000 200 40 | sed "s|}|, \"merge\": \"$m\"}|"
done; done
