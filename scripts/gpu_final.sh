# Final round-2 evidence in one call: the evidence pipeline and the sweeps
# (compute-sanitizer is closed on this pool: scripts/gpu_sanitize.sh when it reopens)
TAG=r02 bash scripts/gpu_evidence.sh
TAG=r02 SWEEPS="long-cot high-concurrency groups" bash scripts/gpu_sweeps.sh
TAG=wl bash scripts/gpu_prof_workloads.sh
