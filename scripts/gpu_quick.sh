timeout 300 python scripts/cfg5_warm.py
CUDA_MODULE_LOADING=EAGER timeout 300 python scripts/cfg5_warm.py
timeout 300 python scripts/cfg5_warm.py
CUDA_MODULE_LOADING=EAGER timeout 300 python scripts/cfg5_warm.py
