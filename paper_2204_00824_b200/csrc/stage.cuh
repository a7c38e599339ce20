// Row gather + distance evaluation shared by the search kernels.
//
// A warp evaluates up to 32 candidate rows at once: lane j owns candidate j.  The
// rows are first staged in the warp's shared-memory slab (32 slots of `dch`+4
// floats: the odd 16-byte pitch makes lane j's LDS.128 of slot j conflict-free),
// then every lane reduces its own slot.
//
// Staging paths (compile-time):
//   kStageLdgsts  cp.async.cg 16-byte copies, one coalesced 512 B row per warp
//                 instruction (lane l moves bytes [16l, 16l+16) of the row);
// Rows are compacted into `slots` slots (fewer slots = less shared memory per
// warp = more resident warps, at the cost of more gather rounds).
//   kStageTma     one cp.async.bulk (TMA, UBLKCP) per row, completion counted on
//                 the warp's mbarrier.
//   kStageG4      TMA tile::gather4 tensor copies: four rows (any row ids) per
//                 instruction through a 2-D tensor map of the vectors (box {dch+4, 1};
//                 the 4 columns past a 128-float row are out of bounds and zero
//                 filled, which gives the padded slot pitch).  A tensor copy needs a
//                 128-byte aligned destination, so the slots sit in groups of 4 at a
//                 gpitch = round_up(4 (dch+4), 32) float stride.  32 rows: 8 issues
//                 instead of 32 (tools/micro/gather4_probe.cu: 1128 vs 2251 cycles
//                 from issue to completion, L2-warm).  Rows of at most 128 floats.
// Distances:
//   exact  the reference's order (vectors.hpp:36-49): acc = ((0+t0)+t1)+..., with
//          t_i = (q_i - r_i)^2 rounded separately — packed FADD2/FMUL2 (f32x2, one
//          rounding per element, so still bit-identical) for the sub/mul, scalar
//          sequential FADD for the sum.
//   fast   FFMA2 into two interleaved partial sums (even/odd dims) — different
//          rounding, shorter dependency chain; only recall-level parity applies.
#pragma once

#include "common.cuh"

namespace tsdg_dev {

enum StageKind { kStageLdgsts = 0, kStageTma = 1, kStageG4 = 2 };

struct WarpStage {
    float* sq;      // query, ld floats (zero padded)
    float* stage;   // 32 x (dch + 4)
    uint64_t* bar;  // TMA path
    uint32_t parity;
    uint32_t* rowid;  // LDGSTS / gather4 paths: row id per slot (32), or nullptr (then __fns)
};

struct Geom {
    const float* vec;
    uint32_t ld, d, dch;
    uint32_t slots;  // shared-memory row slots per warp (1..32)
    uint32_t pitch;  // floats between slots (0: dch + 4, an odd number of 16-byte units)
    const void* tmap;  // kStageG4: the vectors' tensor map (global memory), else unused
    uint32_t gpitch;   // kStageG4: floats between 4-slot groups
};

// Slot s of a warp's staging slab.
template <int STAGE>
__device__ __forceinline__ float* slot_ptr(float* stage, const Geom& g, uint32_t pitch, uint32_t s) {
    return STAGE == kStageG4 ? stage + (s >> 2) * g.gpitch + (s & 3u) * pitch : stage + s * pitch;
}

// tile::gather4: rows r0..r3 (columns c0 .. c0 + box) of the tensor map into four
// consecutive boxes at dst (128-byte aligned), completion counted on bar.
__device__ __forceinline__ void bulk_gather4(void* dst, const void* tmap, uint32_t c0, uint32_t r0,
                                             uint32_t r1, uint32_t r2, uint32_t r3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_addr(dst)),
        "l"(tmap), "r"(smem_addr(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}

// Issue the gather4 copies of `cnt` rows whose ids are in rowid[0, cnt) (slot r <- row
// rowid[r]); a partial last group repeats its first row.  Lane 0 arms the barrier.
__device__ __forceinline__ void g4_issue(WarpStage& w, const Geom& g, uint32_t cnt, int lane) {
    const uint32_t pitch = g.dch + 4;
    const uint32_t ng = (cnt + 3) >> 2;
    if (lane == 0) mbar_arrive_expect_tx(w.bar, ng * 16u * pitch);
    __syncwarp();
    if ((uint32_t)lane < ng) {
        const uint32_t b = 4u * (uint32_t)lane;
        const uint32_t r0 = w.rowid[b];
        const uint32_t r1 = b + 1 < cnt ? w.rowid[b + 1] : r0;
        const uint32_t r2 = b + 2 < cnt ? w.rowid[b + 2] : r0;
        const uint32_t r3 = b + 3 < cnt ? w.rowid[b + 3] : r0;
        bulk_gather4(w.stage + (size_t)lane * g.gpitch, g.tmap, 0, r0, r1, r2, r3, w.bar);
    }
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ unsigned long long f2_pack(float x, float y) {
    return (unsigned long long)__float_as_uint(x) | ((unsigned long long)__float_as_uint(y) << 32);
}
__device__ __forceinline__ float f2_lo(unsigned long long v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float f2_hi(unsigned long long v) {
    return __uint_as_float((uint32_t)(v >> 32));
}
__device__ __forceinline__ unsigned long long f2_sub(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long f2_mul(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long f2_fma(unsigned long long a, unsigned long long b,
                                                     unsigned long long c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// Exact: acc continues the reference's sequential sum over 4 more dims.  Operands
// arrive as packed f32 pairs straight from LDS.128 (ulonglong2), so the paired
// FADD2/FMUL2 need no register shuffling.
template <int METRIC>
__device__ __forceinline__ float acc4_exact2(float acc, ulonglong2 q, ulonglong2 r) {
    unsigned long long t01, t23;
    if (METRIC == 0) {
        const unsigned long long d01 = f2_sub(q.x, r.x), d23 = f2_sub(q.y, r.y);
        t01 = f2_mul(d01, d01);
        t23 = f2_mul(d23, d23);
    } else {
        t01 = f2_mul(q.x, r.x);
        t23 = f2_mul(q.y, r.y);
    }
    acc = __fadd_rn(acc, f2_lo(t01));
    acc = __fadd_rn(acc, f2_hi(t01));
    acc = __fadd_rn(acc, f2_lo(t23));
    acc = __fadd_rn(acc, f2_hi(t23));
    return acc;
}

// Fast: two packed accumulators (even/odd dims).
template <int METRIC>
__device__ __forceinline__ unsigned long long acc4_fast(unsigned long long acc, ulonglong2 q,
                                                        ulonglong2 r) {
    if (METRIC == 0) {
        const unsigned long long d01 = f2_sub(q.x, r.x), d23 = f2_sub(q.y, r.y);
        acc = f2_fma(d01, d01, acc);
        acc = f2_fma(d23, d23, acc);
    } else {
        acc = f2_fma(q.x, r.x, acc);
        acc = f2_fma(q.y, r.y, acc);
    }
    return acc;
}

// Sum over quads [q0, q1) of one staged row; full unroll for the d = 128 case.
template <int METRIC, bool FAST>
__device__ __forceinline__ void row_quads(const float* srow, const float* sq, uint32_t q0,
                                          uint32_t q1, float& acc, unsigned long long& acc2) {
    const ulonglong2* r2 = reinterpret_cast<const ulonglong2*>(srow);
    const ulonglong2* q2 = reinterpret_cast<const ulonglong2*>(sq);
    if (q0 == 0 && q1 == 32) {
#pragma unroll
        for (uint32_t i = 0; i < 32; ++i) {
            if (FAST) acc2 = acc4_fast<METRIC>(acc2, q2[i], r2[i]);
            else acc = acc4_exact2<METRIC>(acc, q2[i], r2[i]);
        }
    } else if (q1 - q0 == 8) {
#pragma unroll
        for (uint32_t i = 0; i < 8; ++i) {
            if (FAST) acc2 = acc4_fast<METRIC>(acc2, q2[q0 + i], r2[q0 + i]);
            else acc = acc4_exact2<METRIC>(acc, q2[q0 + i], r2[q0 + i]);
        }
    } else if (q1 - q0 == 16) {
#pragma unroll
        for (uint32_t i = 0; i < 16; ++i) {
            if (FAST) acc2 = acc4_fast<METRIC>(acc2, q2[q0 + i], r2[q0 + i]);
            else acc = acc4_exact2<METRIC>(acc, q2[q0 + i], r2[q0 + i]);
        }
    } else {
#pragma unroll 4
        for (uint32_t i = q0; i < q1; ++i) {
            if (FAST) acc2 = acc4_fast<METRIC>(acc2, q2[i], r2[i]);
            else acc = acc4_exact2<METRIC>(acc, q2[i], r2[i]);
        }
    }
}

// Stage the rows of the lanes in `need` (row id e per lane) and return each such
// lane's distance to the staged query (+inf for the others).  The needed rows are
// processed in rounds of g.slots (<= 32) shared-memory slots: the r-th needed row
// (lane order) goes to slot r mod slots and is reduced by lane r mod slots; the
// distance is shuffled back to the lane that owns the edge.
template <int METRIC, bool FAST, int STAGE>
__device__ __forceinline__ float gather_eval(WarpStage& w, const Geom& g, bool need, uint32_t e,
                                             int lane) {
    const float kInf = __int_as_float(0x7f800000);
    const unsigned nm = __ballot_sync(kFull, need);
    if (nm == 0) return kInf;
    PH_DECL
    const uint32_t pitch = g.pitch ? g.pitch : g.dch + 4;
    const uint32_t cnt = __popc(nm);
    const uint32_t rank = __popc(nm & ((1u << lane) - 1u));
    const float* row_src = g.vec + (size_t)(need ? e : 0) * g.ld;
    float result = kInf;
    for (uint32_t r0 = 0; r0 < cnt; r0 += g.slots) {
        const uint32_t nr = min(g.slots, cnt - r0);
        const bool mine_round = need && rank >= r0 && rank < r0 + nr;
        const uint32_t slot = rank - r0;
        // fast mode with <= 16 slots: lanes l and l+16 reduce the two halves of slot l
        const bool split = FAST && g.slots <= 16;
        const uint32_t cslot = split ? ((uint32_t)lane & 15u) : (uint32_t)lane;
        const bool half = split && lane >= 16;
        const bool computes = cslot < nr;
        const float* srow = slot_ptr<STAGE>(w.stage, g, pitch, cslot);  // slot reduced by this lane
        float acc = 0.0f;
        unsigned long long acc2 = 0ull;
        for (uint32_t c0 = 0; c0 < g.ld; c0 += g.dch) {
            const uint32_t cw = min(g.dch, g.ld - c0);  // floats this round, multiple of 4
            if (STAGE == kStageG4) {  // whole rows (ld <= dch): one chunk
                __syncwarp();  // the previous round's readers of rowid / the slots are done
                if (mine_round) w.rowid[slot] = e;
                fence_proxy_async_smem();
                __syncwarp();
                g4_issue(w, g, nr, lane);
                mbar_wait(w.bar, w.parity);
                w.parity ^= 1u;
            } else if (STAGE == kStageTma) {
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive_expect_tx(w.bar, nr * cw * 4u);
                __syncwarp();
                if (mine_round) bulk_g2s(w.stage + slot * pitch, row_src + c0, cw * 4u, w.bar);
                mbar_wait(w.bar, w.parity);
                w.parity ^= 1u;
                PH_MARK(3)
            } else {
                __syncwarp();
                const uint32_t nvec = cw >> 2;             // 16-byte pieces per row
                const uint32_t rpi = 32u / nvec;           // rows per warp instruction
                const uint32_t sub = (uint32_t)lane / nvec, piece = (uint32_t)lane % nvec;
                if (w.rowid) {
                    // owners publish their row ids by slot; copiers read them back (a
                    // broadcast LDS) instead of searching the ballot for the owner lane
                    if (c0 == 0 && mine_round) w.rowid[slot] = e;
                    __syncwarp();
                    for (uint32_t t = 0; t < nr; t += rpi) {
                        const uint32_t row = t + sub;
                        if (sub < rpi && row < nr)
                            cp_async16(w.stage + row * pitch + piece * 4,
                                       g.vec + (size_t)w.rowid[row] * g.ld + c0 + piece * 4);
                    }
                } else {
                    for (uint32_t t = 0; t < nr; t += rpi) {
                        const uint32_t want = r0 + t + sub;  // rank of the row this lane moves
                        const bool act = sub < rpi && t + sub < nr;
                        const int src = act ? __fns(nm, 0, (int)want + 1) : 0;
                        const uint32_t er = __shfl_sync(kFull, e, src);
                        if (act)
                            cp_async16(w.stage + (t + sub) * pitch + piece * 4,
                                       g.vec + (size_t)er * g.ld + c0 + piece * 4);
                    }
                }
                cp_async_wait_all();
                __syncwarp();
            }
            if (computes && c0 < g.d) {
                const uint32_t lim = min(cw, g.d - c0);
                const uint32_t quads = lim >> 2;
                // fast mode: two lanes per slot when slots <= 16 (halves of the row)
                uint32_t qa = 0, qb = quads;
                if (FAST && split) {
                    const uint32_t h = quads >> 1;
                    qa = half ? h : 0;
                    qb = half ? quads : h;
                }
                row_quads<METRIC, FAST>(srow, w.sq + c0, qa, qb, acc, acc2);
                if (!(FAST && split && half)) {
                    for (uint32_t i = quads * 4; i < lim; ++i) {
                        const float qv = w.sq[c0 + i], rv = srow[i];
                        if (FAST) {
                            if (METRIC == 0) {
                                const float df = qv - rv;
                                acc = fmaf(df, df, acc);
                            } else {
                                acc = fmaf(qv, rv, acc);
                            }
                        } else {
                            acc = acc_exact<METRIC>(acc, qv, rv);
                        }
                    }
                }
            }
        }
        float dist;
        if (FAST) {
            float part = f2_lo(acc2) + f2_hi(acc2) + acc;
            if (split) part += __shfl_xor_sync(kFull, part, 16);
            dist = finish_exact<METRIC>(part);
        } else {
            dist = finish_exact<METRIC>(acc);
        }
        const float got = __shfl_sync(kFull, dist, (int)(slot & 31u));
        PH_MARK(4)
        if (mine_round) result = got;
    }
    return result;
}

// Split form of gather_eval for one round with whole rows (TMA staging, rows of at
// most dch floats, at most `slots` needed rows): gather_issue starts the copies of the
// needed rows (rank r -> slot r), gather_complete waits for them and returns each
// needed lane's distance.  Lets a kernel put a gather in flight ahead of the work
// that precedes its use (greedy_cta_kernel: the next hop's rows during merge_halves).
__device__ __forceinline__ void gather_issue(WarpStage& w, const Geom& g, bool need, uint32_t e,
                                             int lane) {
    const unsigned nm = __ballot_sync(kFull, need);
    if (nm == 0) return;
    const uint32_t pitch = g.pitch ? g.pitch : g.dch + 4;
    const uint32_t rank = __popc(nm & ((1u << lane) - 1u));
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive_expect_tx(w.bar, __popc(nm) * g.ld * 4u);
    __syncwarp();
    if (need) bulk_g2s(w.stage + rank * pitch, g.vec + (size_t)e * g.ld, g.ld * 4u, w.bar);
}

// LDGSTS form of gather_issue (rows of at most 128 floats, w.rowid set): the needed
// lanes publish their row ids by rank, then every lane copies 16-byte pieces with
// cp.async (one coalesced row per warp instruction at d = 128) — no per-row TMA
// request, which the greedy hop found issue-bound (~30 cycles per 512-B row).
__device__ __forceinline__ void gather_issue_ldgsts(WarpStage& w, const Geom& g, bool need,
                                                    uint32_t e, int lane) {
    const unsigned nm = __ballot_sync(kFull, need);
    if (nm == 0) return;
    const uint32_t pitch = g.pitch ? g.pitch : g.dch + 4;
    const uint32_t cnt = __popc(nm);
    __syncwarp();  // the slots' previous rows have been consumed
    if (need) w.rowid[__popc(nm & ((1u << lane) - 1u))] = e;
    __syncwarp();
    const uint32_t nvec = g.ld >> 2, rpi = 32u / nvec;
    const uint32_t sub = (uint32_t)lane / nvec, piece = (uint32_t)lane % nvec;
    if (nvec == 32) {
        // one 512-B row per warp instruction; the row ids come from registers
        // (shuffles), so successive copies do not wait on each other: no "memory"
        // clobber between them (the staging slots are read only after the
        // cp.async.wait_group in gather_complete, which carries one)
        const uint32_t rid = w.rowid[lane];
        const float* src = g.vec + piece * 4;
        float* dst = w.stage + piece * 4;
#pragma unroll 8
        for (uint32_t r = 0; r < cnt; ++r) {
            const uint32_t id = __shfl_sync(kFull, rid, (int)r);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst + r * pitch)),
                         "l"(src + (size_t)id * g.ld));
        }
    } else {
        for (uint32_t t = 0; t < cnt; t += rpi) {
            const uint32_t row = t + sub;
            if (sub < rpi && row < cnt)
                cp_async16(w.stage + row * pitch + piece * 4, g.vec + (size_t)w.rowid[row] * g.ld + piece * 4);
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}
// gather4 form of gather_issue (rows of at most dch floats, w.rowid set).
__device__ __forceinline__ void gather_issue_g4(WarpStage& w, const Geom& g, bool need, uint32_t e,
                                                int lane) {
    const unsigned nm = __ballot_sync(kFull, need);
    if (nm == 0) return;
    __syncwarp();  // the slots' previous rows and rowid have been consumed
    if (need) w.rowid[__popc(nm & ((1u << lane) - 1u))] = e;
    fence_proxy_async_smem();
    __syncwarp();
    g4_issue(w, g, __popc(nm), lane);
}
template <int STAGE>
__device__ __forceinline__ void gather_issue_s(WarpStage& w, const Geom& g, bool need, uint32_t e,
                                               int lane) {
    if (STAGE == kStageTma) gather_issue(w, g, need, e, lane);
    else if (STAGE == kStageG4) gather_issue_g4(w, g, need, e, lane);
    else gather_issue_ldgsts(w, g, need, e, lane);
}

template <int METRIC, bool FAST, int STAGE = kStageTma>
__device__ __forceinline__ float gather_complete(WarpStage& w, const Geom& g, bool need, int lane) {
    const float kInf = __int_as_float(0x7f800000);
    const unsigned nm = __ballot_sync(kFull, need);
    if (nm == 0) return kInf;
    const uint32_t pitch = g.pitch ? g.pitch : g.dch + 4;
    const uint32_t cnt = __popc(nm);
    const uint32_t rank = __popc(nm & ((1u << lane) - 1u));
    if (STAGE != kStageLdgsts) {
        mbar_wait(w.bar, w.parity);
        w.parity ^= 1u;
    } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
    }
    float dist = kInf;
    if ((uint32_t)lane < cnt) {  // lane r reduces slot r, in the reference's order
        const float* srow = slot_ptr<STAGE>(w.stage, g, pitch, (uint32_t)lane);
        float acc = 0.0f;
        unsigned long long acc2 = 0ull;
        const uint32_t quads = g.d >> 2;
        row_quads<METRIC, FAST>(srow, w.sq, 0, quads, acc, acc2);
        for (uint32_t i = quads * 4; i < g.d; ++i) {
            if (FAST) {
                const float df = w.sq[i] - srow[i];
                acc = METRIC == 0 ? fmaf(df, df, acc) : fmaf(w.sq[i], srow[i], acc);
            } else {
                acc = acc_exact<METRIC>(acc, w.sq[i], srow[i]);
            }
        }
        dist = FAST ? finish_exact<METRIC>(f2_lo(acc2) + f2_hi(acc2) + acc) : finish_exact<METRIC>(acc);
    }
    const float got = __shfl_sync(kFull, dist, (int)(rank & 31u));
    __syncwarp();
    return need ? got : kInf;
}

}  // namespace tsdg_dev
