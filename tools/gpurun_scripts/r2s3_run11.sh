timeout 600 python tools/restore_profile.py cfg1 > gpurun_out/s3_restore_profile_cfg1.log 2>&1
