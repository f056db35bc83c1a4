# Final round-2 evidence in one call: the evidence pipeline, the sweeps, the sanitizers
TAG=r02 bash scripts/gpu_evidence.sh
TAG=r02 SWEEPS="long-cot high-concurrency groups" bash scripts/gpu_sweeps.sh
TAG=r02 bash scripts/gpu_sanitize.sh
