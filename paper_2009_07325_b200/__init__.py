"""B200-native gIM/IMM hot path (arXiv 2009.07325): RR-set sampling + greedy max-coverage
NodeSelection + the IMM theta loop, behind the C ABI of include/gim.h (libgim.so, sm_100a)."""
from .gim import (Gim, GimError, ImmResult, IC, LT, W_EXPLICIT, W_WC, W_UNIFORM,  # noqa: F401
                  OPT_FORCE_GIANT, OPT_QUEUE_CAP, OPT_PROFILE, OPT_STAGING_CAP, OPT_SELECT_GRAPH, OPT_INV_SEGMENTS, OPT_ARGMAX_CAND, OPT_IC_LANE, OPT_SPECULATE, OPT_MB_CHAINS, OPT_PDL, OPT_GIANT_NT, OPT_FRESH_FINAL, OPT_SELECT_PERSISTENT, OPT_SKIP, OPT_SPILL, OPT_SELECT_FUSED, OPT_FUSED_CTAS, OPT_FORCE_COLLECTIVES, OPT_GIANT_SHARED, OPT_SKIP_LANE_CAP, OPT_SELECT_COOP,
                  OPT_IMM_EARLY_EXIT, OPT_INV_PASSES, OPT_L2_PERSIST, OPT_SELECT_CTA, OPT_INV_SORT, OPT_CHUNK, OPT_SELECT_CLUSTER, OPT_IMM_LOOKAHEAD, load_library,
                  torch_allreduce, torch_allgather, torch_reducescatter, shard_slice, SIGNATURES, LIB_PATH,
                  nccl_unique_id, setup_nccl)
