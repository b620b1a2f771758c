for cfg in "1 1 1" "1 1 0" "1 0 0" "1 0 1" "0 1 0" "0 0 0"; do
  set -- $cfg
  echo "RCB=$1 SPLIT=$2 SORT=$3"
  for d in "20 20 21" "15 15 16"; do RAFEM_CL_RCB=$1 RAFEM_CL_SPLIT=$2 RAFEM_CL_SORT=$3 timeout 60 python scripts/cluster_phase.py $d | tail -1; done
done
