set -x
python tools/sanitize_seam.py > gpurun_out/q2_seam_plain.log 2>&1
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_seam.py > gpurun_out/q2_seam_memcheck.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_seam.py > gpurun_out/q2_seam_racecheck.log 2>&1
timeout 600 compute-sanitizer --tool synccheck python tools/sanitize_seam.py > gpurun_out/q2_seam_synccheck.log 2>&1
python tools/host_overhead.py 1024,32,1 65536,64,1 > gpurun_out/q2_host.log 2>&1
timeout 1200 python tools/stress.py 80 2 > gpurun_out/q2_stress.log 2>&1
