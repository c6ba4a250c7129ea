cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_configs.py -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_cfg.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_cfg.log
