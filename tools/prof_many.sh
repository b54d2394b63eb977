# Role-loop profiles of many-expert launches (tools/ktiming.py, MESW_PROFILE build)
mkdir -p gpurun_out
MESW_PROFILE=1 python build.py --force > /dev/null 2>&1
cd tools
for cfg in "4 64" "8 128" "16 128" "8 64"; do
  set -- $cfg
  echo "=== E=$1 B=$2"
  ALIGNED=1 timeout 120 python ktiming.py 4096 14336 $1 $2 2>&1 | grep -v "jobs (\|unit ends\|chunk ends"
done
