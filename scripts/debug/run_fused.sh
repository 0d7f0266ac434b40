timeout 60 python scripts/debug/fused_short.py 51277 300; echo rc=$?
timeout 60 python scripts/debug/fused_short.py 51277 30; echo rc=$?
timeout 60 python scripts/debug/fused_short.py 2048 300; echo rc=$?
timeout 120 compute-sanitizer --tool memcheck python scripts/debug/fused_short.py 2048 300 2>&1 | tail -20; echo rc=$?
