#!/usr/bin/env bash
# Offline preparation of every benchmark / parity dataset under data/ (inputs only,
# never timed).  Needs oracle/_ref (the reference compiled from /root/reference by
# __graft_entry__.build()).  data/ is git-ignored; the packed graphs
# (graph.pk) travel to the GPU box with the gpurun snapshot, the unpacked
# graph.tsdg files are rebuilt there byte-identically (tools/graph_pack.py).
#
#   bash tools/prepare_data.sh [c2] [c1] [c5s] [c4]     (default: all, in that order)
set -euo pipefail
cd "$(dirname "$0")/.."
want=("$@")
[ ${#want[@]} -eq 0 ] && want=(c2 c1 c5s c4)
for w in "${want[@]}"; do
  case "$w" in
    c2)  # SIFT1M shape: 1M x 128, nn_descent k=64 (SURVEY.md §8(d) recipe 3)
      [ -f data/c2_lowlid_1m/gt.u32 ] || python tools/make_dataset.py --name c2_lowlid_1m \
        --kind lowlid --n 1000000 --nq 10000 --d 128 --latent 16 --builder nndescent --knn-k 64 --iters 5
      [ -f data/c2_lowlid_1m/graph.pk ] || python tools/graph_pack.py c2_lowlid_1m ;;
    c1)  # CPU-runnable config: 100K x 128, brute-force k=100 graph, 1K queries
      [ -f data/c1_lowlid_100k/gt.u32 ] || python tools/make_dataset.py --name c1_lowlid_100k \
        --kind lowlid --n 100000 --nq 1000 --d 128 --latent 16 --builder brute --knn-k 100
      [ -f data/c1_lowlid_100k/graph.pk ] || python tools/graph_pack.py c1_lowlid_100k ;;
    c5s) # Deep100M shape scaled: 2M x 96 in 8 shards, one TSDG per shard
      [ -f data/c5s_lowlid_2m_96/meta.json ] || python tools/make_sharded.py --name c5s_lowlid_2m_96 \
        --n 2000000 --nq 10000 --d 96 --latent 16 --shards 8 --knn-k 32 --iters 5 ;;
    c4)  # GIST1M shape: 1M x 960 (latent 26), nn_descent k=64
      [ -f data/c4_lowlid_1m_960/gt.u32 ] || python tools/make_dataset.py --name c4_lowlid_1m_960 \
        --kind lowlid --n 1000000 --nq 10000 --d 960 --latent 26 --builder nndescent --knn-k 64 --iters 5
      [ -f data/c4_lowlid_1m_960/graph.pk ] || python tools/graph_pack.py c4_lowlid_1m_960 ;;
    *) echo "unknown dataset $w" >&2; exit 1 ;;
  esac
done
