bash tools/profile_r02.sh > gpurun_out/profile.log 2>&1
