# A/B of an environment switch: bash scripts/ab_env.sh "<configs>" VAR "v1 v2 ..."  (results in gpurun_out/ab.log)
mkdir -p gpurun_out; : > gpurun_out/ab.log
cfgs=$1; var=$2; vals=$3
for rep in 1 2; do for cfg in $cfgs; do for v in $vals; do
  echo "$var=$v" >> gpurun_out/ab.log
  env $var=$v timeout 300 python scripts/ab_c5.py $cfg 10 >> gpurun_out/ab.log 2>&1
done; done; done
