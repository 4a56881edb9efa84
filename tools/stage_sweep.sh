for kb in 48 56 64 80; do MPID_PASS_STAGE_KB=$kb python tools/pass_tune.py 4 5 6; done
