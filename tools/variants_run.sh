# A/B timing of build variants / env switches on the C2 PCG round (tools/profile_pcg.py)
cfg=${CFG:-c2}
for v in "$@"; do
  case $v in
    env:*) e=${v#env:}; n=$v; unset HFB200_LIB; export $e ;;
    lib:*) n=$v; export HFB200_LIB=$PWD/paper_1811_07717_b200/_lib/variants/libhfb200_${v#lib:}.so ;;
    *) n=cur; unset HFB200_LIB ;;
  esac
  echo "$n $(timeout 300 python tools/profile_pcg.py --config $cfg --rounds 20 2>&1 | grep -o "'kernels'.*" | cut -c1-200)"
  [ "${v#env:}" != "$v" ] && unset ${e%%=*}
done
