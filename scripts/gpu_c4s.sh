timeout 600 python scripts/cfg4_steps.py batch 2>/dev/null | tail -12
timeout 600 python scripts/cfg4_steps.py single 2>/dev/null | tail -12
