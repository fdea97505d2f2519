# Plumbing check of the N > 1 bench path on ONE GPU (all ranks share it, bands staged
# through the host over gloo: never a timing).  The residual history of every N must
# equal the single-domain run of the same global problem:
#   c4 (strong, 256^2, n_a = 16) at N = 1, 2, 4, 8;
#   c5w (weak: (512 N) x 512, n_a = 4, 7 groups) at N = 2, 4, 8 vs --slabs N on 1 rank;
#   c5 (strong: 1024^2, 7 groups, n_a = 2) at N = 4, 8 vs N = 1.
set -x
mkdir -p gpurun_out
run() {   # tag nproc args...
  local tag=$1 n=$2; shift 2
  if [ "$n" = 1 ]; then
    timeout 900 python bench.py "$@" > gpurun_out/dd_$tag.log 2>&1
  else
    CSN_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 \
      --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) \
      bench.py --gpus $n "$@" > gpurun_out/dd_$tag.log 2>&1
  fi
}
C4="--nx 256 --steps 6 --warmup 3 --no-cpu --no-e2e --no-extra"
run c4_n1 1 $C4
for n in 2 4 8; do run c4_n$n $n $C4; done
W="--config c5w --na 4 --steps 3 --warmup 3 --no-cpu --no-e2e --no-extra"
for n in 2 4 8; do run c5w_ref$n 1 $W --slabs $n; run c5w_n$n $n $W; done
# c5 (strong, 1024^2, 7 groups) at n_a = 2: N = 4, 8 vs N = 1
S="--config c5 --na 2 --steps 3 --warmup 3 --no-cpu --no-e2e --no-extra"
run c5_n1 1 $S
for n in 4 8; do run c5_n$n $n $S; done
python - <<'PY'
import json
def hist(tag):
    t = open(f"gpurun_out/dd_{tag}.log").read().strip().splitlines()
    d = [json.loads(l) for l in t if l.startswith("{")][-1]
    return d["residual_history"], d.get("k_history")
out = []
h1, _ = hist("c4_n1")
for n in (2, 4, 8):
    h, _ = hist(f"c4_n{n}")
    out.append(f"c4 N={n}: max rel diff of the residual history vs N=1: "
               f"{max(abs(a / b - 1) for a, b in zip(h, h1)):.2e} ({len(h)} cycles)")
for n in (2, 4, 8):
    h, k = hist(f"c5w_n{n}")
    r, kr = hist(f"c5w_ref{n}")
    out.append(f"c5w N={n} ((512 N) x 512): residual history vs single-domain "
               f"{max(abs(a / b - 1) for a, b in zip(h, r)):.2e}, k history "
               f"{max(abs(a / b - 1) for a, b in zip(k, kr)):.2e}")
h1, k1 = hist("c5_n1")
for n in (4, 8):
    h, k = hist(f"c5_n{n}")
    out.append(f"c5 N={n} (1024^2, 7 groups, n_a=2): residual history vs N=1 "
               f"{max(abs(a / b - 1) for a, b in zip(h, h1)):.2e}, k history "
               f"{max(abs(a / b - 1) for a, b in zip(k, k1)):.2e}")
open("gpurun_out/dd_plumbing_summary.txt", "w").write("\n".join(out) + "\n")
print("\n".join(out))
PY
