for cfg in "default::" "v4pf296:v4:296" "v4pf148:v4:148" "v4pf600:v4:600" "v4pf0:v4:0"; do
  name=${cfg%%:*}; rest=${cfg#*:}; impl=${rest%%:*}; pf=${rest#*:}
  env_args=""
  [ -n "$impl" ] && env_args="$env_args QAOA_SWEEP_IMPL=$impl"
  [ -n "$pf" ] && env_args="$env_args QAOA_PF_DIST=$pf"
  env $env_args timeout 200 python bench.py --steps 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pf_$name.log 2>&1
done
