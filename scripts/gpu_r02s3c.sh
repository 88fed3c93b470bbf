# hub table A/B at T: table size and CTA shape
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() { # name env...
  n=$1; shift
  env "$@" timeout 600 python scripts/round_profile.py --config T --reps 1 > gpurun_out/s3c_$n.txt 2>&1
  echo "$n: $(head -1 gpurun_out/s3c_$n.txt | grep -o "'rounds': [0-9.]*\|'edgelist': [0-9.]*\|'init': [0-9.]*" | tr '\n' ' ') | r1-4,11,12: $(sed -n 3,6p gpurun_out/s3c_$n.txt | awk '{print $5}' | tr '\n' ' ') $(sed -n 13,14p gpurun_out/s3c_$n.txt | awk '{print $5}' | tr '\n' ' ')"
}
run nohub PICO_HUB_MAX=0
run nohub1024 PICO_HUB_MAX=0 PICO_ROUNDS_1024=1
run hub8k PICO_HUB_MAX=8192
run hub24k PICO_HUB_MAX=24576
run hub48k PICO_HUB_MAX=49152
