bash tools/profile_compact.sh C3 r01f > /dev/null 2>&1
bash tools/profile_compact.sh C2 r01f > /dev/null 2>&1
ls gpurun_out/prof_r01f_C3 gpurun_out/prof_r01f_C2
