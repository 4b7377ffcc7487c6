// merge.cuh — per-queue merge of the partial pass's CTA rows (K7 + K8).
//
// One CTA per queue (looping when there are more queues than CTAs) merges the
// candidate rows into the exact per-queue top-k, member count, FIFO head and
// max score; when the partial pass found gap-falling lengths it first runs
// Alg. 2 (App. D) over the gap list sorted by global id (R22), and
// the last CTA to finish picks Alg. 1's ArgMax queue.
#include <cfloat>
#include <climits>
#pragma once
#include "tick.cuh"

namespace ewsjf {
// merge-phase timestamps (EWSJF_PHASES): max over CTAs of slot x of the per-CTA debug row
#define MDBG(slot_)                                                                                    \
    do {                                                                                           \
        if (A.dbg && threadIdx.x == 0) {                                                           \
            unsigned long long t_;                                                                 \
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_));                                  \
            atomicMax(&A.dbg[blockIdx.x * kDbgStride + (slot_)], t_);                                        \
        }                                                                                          \
    } while (0)
__host__ __device__ inline int64_t al16m(int64_t x) { return (x + 15) & ~(int64_t)15; }

// ------------------------------------------------------------------ merge ---
constexpr int kMThreads = 512;
constexpr int kRankMax = 512;         // survivors rank-sorted at the end

struct MergeSmem {
    int64_t uni, psp, tables, rowoff, surv, ssp, misc, total;
    int esmem;
};
__host__ __device__ inline MergeSmem merge_layout(int in_mode) {
    MergeSmem L;
    const int64_t uni_bytes = 131072;   // gap-phase sort keys | select-phase candidate pool
    L.esmem = in_mode == MERGE_IN_ROWS ? 16384 : 10240;
    int64_t o = 0;
    L.uni = o;    o += uni_bytes;
    L.psp = in_mode == MERGE_IN_ROWS ? 0 : 8 * (int64_t)L.esmem;   // payloads after the keys (exchange)
    L.tables = o; o = al16m(o + 4 * 6 * kMaxSlots);
    L.rowoff = o; o = al16m(o + 4 * 1025);
    L.surv = o;   o = al16m(o + 8 * kRankMax);
    L.ssp = o;    o = al16m(o + 4 * kRankMax);
    L.misc = o;   o = al16m(o + 256);
    L.total = o;
    return L;
}

struct MMisc {
    unsigned long long maxk;
    unsigned long long sec;
    unsigned long long members;
    int cnt[3];
    int nfinal, nbub, ndrop, nmine, pn, nsurv, is_last, gexc;
    float sec_sp;
    unsigned cmin;      // Alg. 2 epoch: lowest creator gid
    int vcre;           // ... its gap-list index
    int nkeep;          // ... requests classified again next epoch
};

// A7 for a bubble (device side, same canonical fp64 expression as the host).
static __device__ __forceinline__ void bubble_weights(const double* th, double L, float* wb, float* wu, float* wf) {
    const double b = __dadd_rn(__dmul_rn(th[0], L), th[1]);
    const double u = __dadd_rn(__dmul_rn(th[2], L), th[3]);
    const double f = __dadd_rn(__dmul_rn(th[4], L), th[5]);
    *wb = (float)(b > 0.0 ? b : 0.0);
    *wu = (float)(u > 0.0 ? u : 0.0);
    const float f32 = (float)(f > 0.0 ? f : 0.0);
    *wf = (float)__dmul_rn((double)f32, 0.69314718055994530942);
}

// CTA-wide count of pool keys >= t (one barrier; rotating counters).
template <int NT>
static __device__ __forceinline__ int pool_count_ge(const u64* pool, int n, u64 t, MMisc* M, int it) {
    int c = 0;
    for (int i = threadIdx.x; i < n; i += NT) c += pool[i] >= t;
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&M->cnt[it % 3], c);
    __syncthreads();
    const int total = M->cnt[it % 3];
    if (threadIdx.x == 0) M->cnt[(it + 2) % 3] = 0;
    return total;
}

// Shrink the pool to the keys >= t where K <= #(>= t) <= kRankMax (bisection,
// requires #(>= lo) >= K); survivors are moved to the front.
template <int NT>
static __device__ void pool_shrink(u64* pool, float* psp, int& pn, u64& lo, int K, u64* surv, float* ssp, MMisc* M) {
    const int tid = threadIdx.x;
    u64 mx = 0;
    for (int i = tid; i < pn; i += NT) mx = pool[i] > mx ? pool[i] : mx;
    mx = warp_max_u64(mx);
    __syncthreads();
    if (tid == 0) { M->maxk = 0; M->cnt[0] = M->cnt[1] = M->cnt[2] = 0; M->nsurv = 0; }
    __syncthreads();
    if ((tid & 31) == 0 && mx) atomicMax(&M->maxk, mx);
    __syncthreads();
    u64 hi = M->maxk + 1ull;
    int it = 0;
    while (hi - lo > 1ull) {
        const u64 mid = lo + (hi - lo) / 2ull;
        const int c = pool_count_ge<NT>(pool, pn, mid, M, it++);
        if (c >= K) {
            lo = mid;
            if (c <= kRankMax) break;
        } else {
            hi = mid;
        }
    }
    for (int i = tid; i < pn; i += NT) {
        if (pool[i] >= lo) {
            const int p = atomicAdd(&M->nsurv, 1);
            EWSJF_CHECK(p < kRankMax);
            surv[p] = pool[i];
            if (psp) ssp[p] = psp[i];
        }
    }
    __syncthreads();
    pn = M->nsurv;
    for (int i = tid; i < pn; i += NT) {
        pool[i] = surv[i];
        if (psp) psp[i] = ssp[i];
    }
    __syncthreads();
}

template <int IN, int OUT, bool HAS_COST, int NT = kMThreads>
__device__ __forceinline__ void merge_phase(const MergeArgs& A, const Policy& P, unsigned char* smem) {
    const MergeSmem L = merge_layout(IN);
    const int tid = threadIdx.x, lane = tid & 31;
    u64* uni = (u64*)(smem + L.uni);
    float* psp = IN == MERGE_IN_EXCHANGE ? (float*)(smem + L.uni + L.psp) : nullptr;
    int* t_lo = (int*)(smem + L.tables);
    int* t_hi = t_lo + kMaxSlots;
    int* t_slot = t_hi + kMaxSlots;   // position -> internal slot
    int* t_pos = t_slot + kMaxSlots;  // internal slot -> position
    int* t_L = t_pos + kMaxSlots;     // bubble creating length (internal slot >= nq)
    int* t_id = t_L + kMaxSlots;      // internal slot -> stable id
    int* rowoff = (int*)(smem + L.rowoff);
    u64* surv = (u64*)(smem + L.surv);
    float* ssp = (float*)(smem + L.ssp);
    MMisc* M = (MMisc*)(smem + L.misc);
    const int nq = A.nq, K = A.K;
    const ExLayout X = ex_layout(nq, K, A.ex_gap);
    const bool is_score = A.sp.mode == EWSJF_SELECT_SCORE;

    // ---------------- gap list size (virtual index v = position in the concatenation
    // of the gap lists: the single list, or rank 0's entries then rank 1's ...)
    long long graw = 0, gcount = 0;
    if (IN == MERGE_IN_ROWS) {
        graw = (long long)__ldcg(&A.ctr->gap_count);
        gcount = graw < A.gap_cap ? graw : A.gap_cap;
    } else {
        for (int r = 0; r < A.world; r++) {
            const long long c = ((const ExHeader*)(A.ex_in + (int64_t)r * A.ex_bytes))->gap_count;
            graw += c;
            gcount += c < X.gap_cap ? c : X.gap_cap;
        }
    }
    if (gcount > A.gap_cap) gcount = A.gap_cap;
    const bool gap_overflow = graw > gcount;
    auto gap_entry = [&](uint32_t v) -> GapEntry {
        if (IN == MERGE_IN_ROWS) return A.gap[v];
        long long acc = 0;
        int r = 0;
        for (; r < A.world; r++) {
            long long c = ((const ExHeader*)(A.ex_in + (int64_t)r * A.ex_bytes))->gap_count;
            c = c < X.gap_cap ? c : X.gap_cap;
            if ((long long)v < acc + c) break;
            acc += c;
        }
        return ((const GapEntry*)(A.ex_in + (int64_t)r * A.ex_bytes + X.gaps))[v - acc];
    };

    // ---------------- final partition: App. D Alg. 2 over the gap requests in global
    // index order (R22), epoch-parallel and exact.  Requests in index order see the
    // partition unchanged until the first one that creates a bubble; so in each
    // epoch every unresolved request is classified against the current table in
    // parallel (inside a queue / tolerated by a neighbour, R19 / would create a
    // bubble), the lowest-index creator c inserts its bubble (R20), every request
    // before c is final, and after c only those in c's gap and the other pending
    // creators are classified again (a bubble changes nothing outside its gap; a
    // request inside a queue stays there).  At most 256 - nq epochs.  CTA 0 runs it
    // and publishes the table; the other CTAs wait for it.
    for (int i = tid; i < nq; i += NT) {
        t_lo[i] = P.min_len[i]; t_hi[i] = P.max_len[i];
        t_slot[i] = i; t_pos[i] = i; t_id[i] = P.sid[i];
    }
    if (tid == 0) { M->nfinal = nq; M->nbub = 0; M->ndrop = 0; M->nmine = 0; M->gexc = 0; }
    __syncthreads();
    const bool do_gaps = gcount > 0 && OUT != MERGE_OUT_EXCHANGE;
    if (do_gaps && blockIdx.x == 0) {
        unsigned* cmin_s = (unsigned*)&M->cmin;
        int n = nq, nb = 0, nd = 0;
        long long nu = gcount;
        bool first = true;
        int32_t* ucur = A.g_u0;
        int32_t* unext = A.g_u1;
        // classification word: slot (10 bits, 1023 = drop) | class << 10 | gap << 12
        constexpr int kClsIn = 0, kClsTol = 1, kClsNew = 2, kClsDrop = 3;
        unsigned* mincre = (unsigned*)uni;       // [gap index 0..n]: lowest creator gid in that gap (uni is free here)
        for (;;) {
            if (tid == 0) { *cmin_s = 0xffffffffu; M->nkeep = 0; }
            for (int i = tid; i <= n; i += NT) mincre[i] = 0xffffffffu;
            __syncthreads();
            for (long long idx = tid; idx < nu; idx += NT) {
                const uint32_t v = first ? (uint32_t)idx : (uint32_t)ucur[idx];
                const GapEntry g = gap_entry(v);
                const int Lq = g.len;
                int lo = 0, hi = n;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (t_lo[mid] <= Lq) lo = mid + 1; else hi = mid;
                }
                const int i = lo - 1;
                int cls, slot = 1023;
                if (i >= 0 && Lq < t_hi[i]) {
                    cls = kClsIn; slot = t_slot[i];
                } else {
                    const bool hl = i >= 0, hr = i + 1 < n;
                    const long long L64 = Lq;
                    if (hl && 10 * L64 <= 11 * (long long)t_hi[i]) { cls = kClsTol; slot = t_slot[i]; }
                    else if (hr && 10 * L64 >= 9 * (long long)t_lo[i + 1]) { cls = kClsTol; slot = t_slot[i + 1]; }
                    else if (n >= kMaxSlots) cls = kClsDrop;
                    else { cls = kClsNew; atomicMin(cmin_s, g.gid); atomicMin(&mincre[i + 1], g.gid); }
                }
                A.g_res[v] = slot | (cls << 10) | ((i + 1) << 12);
            }
            __syncthreads();
            const unsigned cmin = *cmin_s;
            if (cmin == 0xffffffffu) {            // no creator left: every pending request is final
                for (long long idx = tid; idx < nu; idx += NT) {
                    const uint32_t v = first ? (uint32_t)idx : (uint32_t)ucur[idx];
                    const int r = A.g_res[v];
                    const int slot = r & 1023;
                    A.g_slot[v] = slot == 1023 ? -1 : slot;
                    if (slot == 1023) atomicAdd(&M->ndrop, 1);
                }
                __syncthreads();
                break;
            }
            // the creator (unique gid) inserts its bubble
            for (long long idx = tid; idx < nu; idx += NT) {
                const uint32_t v = first ? (uint32_t)idx : (uint32_t)ucur[idx];
                if (((A.g_res[v] >> 10) & 3) == kClsNew && gap_entry(v).gid == cmin) M->vcre = (int)v;
            }
            __syncthreads();
            const int vc = M->vcre;
            const int cgap = A.g_res[vc] >> 12;       // gap index: between positions cgap-1 and cgap
            if (tid == 0) {
                const int i = cgap - 1;
                const int Lq = gap_entry((uint32_t)vc).len;
                const bool hl = i >= 0, hr = i + 1 < n;
                const long long L64 = Lq;
                const long long lb = hl ? t_hi[i] : 1;
                const long long rb = hr ? t_lo[i + 1] : (1ll << 40);
                const long long avail = rb - lb;
                const long long rg = (long long)A.bubble_width < avail ? (long long)A.bubble_width : avail;
                long long nlo = L64 - rg / 2;
                if (nlo < lb) nlo = lb;
                long long nhi = L64 + (rg + 1) / 2;
                if (nhi > rb) nhi = rb;
                if (nhi > INT_MAX) nhi = INT_MAX;
                for (int p = n; p > i + 1; p--) {
                    t_lo[p] = t_lo[p - 1]; t_hi[p] = t_hi[p - 1]; t_slot[p] = t_slot[p - 1];
                }
                const int ns = nq + nb;
                t_lo[i + 1] = (int)nlo; t_hi[i + 1] = (int)nhi; t_slot[i + 1] = ns;
                t_L[ns] = Lq;
                t_id[ns] = A.next_id + nb;
                if (A.blog) {
                    A.blog->pos[nb] = i + 1; A.blog->lo[nb] = (int)nlo;
                    A.blog->hi[nb] = (int)nhi; A.blog->L[nb] = Lq;
                }
                A.g_slot[vc] = ns;
                M->nfinal = n + 1;
            }
            __syncthreads();
            const int ns = nq + nb;
            n++; nb++;
            // settle: a request before c is final; after c, one inside a queue is final,
            // a creator goes again, and a tolerated one goes again only if some creator
            // precedes it in its own gap (that bubble may become its neighbour)
            for (long long idx = tid; idx < nu; idx += NT) {
                const uint32_t v = first ? (uint32_t)idx : (uint32_t)ucur[idx];
                if ((int)v == vc) continue;
                const int r = A.g_res[v];
                const int cls = (r >> 10) & 3, slot = r & 1023, gp = r >> 12;
                const unsigned gid = gap_entry(v).gid;
                bool keep;
                if (cls == kClsIn || cls == kClsDrop || gid < cmin) keep = false;
                else keep = cls == kClsNew || gid > mincre[gp];
                if (keep) {
                    const int o = atomicAdd(&M->nkeep, 1);
                    EWSJF_CHECK((unsigned long long)o < (unsigned long long)A.gap_cap);
                    unext[o] = (int32_t)v;
                } else {
                    A.g_slot[v] = slot == 1023 ? -1 : slot;
                    if (slot == 1023) atomicAdd(&M->ndrop, 1);
                }
            }
            __syncthreads();
            nu = M->nkeep;
            first = false;
            int32_t* t = ucur; ucur = unext; unext = t;
            (void)ns;
            if (nu == 0) break;
            __syncthreads();
        }
        nd = M->ndrop;
        if (tid == 0) {
            M->nfinal = n; M->nbub = nb;
            A.g_tab[0] = n; A.g_tab[1] = nb; A.g_tab[2] = nd;
        }
        __syncthreads();
        for (int i = tid; i < n; i += NT) {
            A.g_tab[3 + i] = t_lo[i]; A.g_tab[3 + kMaxSlots + i] = t_hi[i]; A.g_tab[3 + 2 * kMaxSlots + i] = t_slot[i];
        }
        for (int i = tid; i < nq + nb; i += NT) {
            A.g_tab[3 + 3 * kMaxSlots + i] = t_L[i]; A.g_tab[3 + 4 * kMaxSlots + i] = t_id[i];
        }
        // qid write-back of this rank's gap requests (stable ids)
        if (A.qid) {
            for (long long e = tid; e < gcount; e += NT) {
                const GapEntry g = gap_entry((uint32_t)e);
                const long long li = (long long)g.gid - (long long)A.gbase;
                if (li >= 0 && li < A.n_local) { const int as = A.g_slot[e]; A.qid[li] = as >= 0 ? t_id[as] : -1; }
            }
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&A.ctr->gap_done), "r"(A.seq) : "memory");
    } else if (do_gaps) {
        if (tid == 0) {
            unsigned v;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&A.ctr->gap_done) : "memory");
                if (v != A.seq) __nanosleep(200);
            } while (v != A.seq);
        }
        __syncthreads();
        const int n = __ldcg(&A.g_tab[0]), nb = __ldcg(&A.g_tab[1]);
        for (int i = tid; i < n; i += NT) {
            t_lo[i] = __ldcg(&A.g_tab[3 + i]); t_hi[i] = __ldcg(&A.g_tab[3 + kMaxSlots + i]);
            t_slot[i] = __ldcg(&A.g_tab[3 + 2 * kMaxSlots + i]);
        }
        for (int i = tid; i < nq + nb; i += NT) {
            t_L[i] = __ldcg(&A.g_tab[3 + 3 * kMaxSlots + i]); t_id[i] = __ldcg(&A.g_tab[3 + 4 * kMaxSlots + i]);
        }
        if (tid == 0) { M->nfinal = n; M->nbub = nb; M->ndrop = __ldcg(&A.g_tab[2]); }
        __syncthreads();
    }
    if (do_gaps) {
        for (int p = tid; p < M->nfinal; p += NT) t_pos[t_slot[p]] = p;
        __syncthreads();
    }
    if (blockIdx.x == 0 && A.blog && tid == 0) A.blog->n = M->nbub;
    const int nfinal = M->nfinal;
    const long long ngap_all = do_gaps ? gcount : 0;   // every gap entry is checked against the slot
    const int nloop = OUT == MERGE_OUT_ROUTE ? 0 : (OUT == MERGE_OUT_EXCHANGE ? nq : nfinal);

    for (int s = blockIdx.x; s < nloop; s += gridDim.x) {
        float wb, wu, wf;
        if (s < nq) { wb = P.wb[s]; wu = P.wu[s]; wf = P.wf[s]; }
        else bubble_weights(A.theta, (double)t_L[s], &wb, &wu, &wf);
        // payload s' of a local-pool request (rows input)
        auto recompute = [&](uint32_t gid) -> float {
            const long long li = (long long)gid - (long long)A.gbase;
            float sp = 0.f;
            if (li >= 0 && li < A.n_local)
                score_sp(__ldg(A.len + li), __ldg(A.arrival + li), HAS_COST ? __ldg(A.cost + li) : 0.f, HAS_COST,
                         A.sp, wb, wu, wf, &sp);
            return sp;
        };
        auto gap_keys = [&](const GapEntry& g, u64& k1, u64& k2, float& sp) -> bool {
            const bool hc = !(g.cost != g.cost);
            const bool ok = score_sp(g.len, g.arrival, hc ? g.cost : 0.f, hc, A.sp, wb, wu, wf, &sp);
            const u64 ks = score_key(sp, g.gid), kf = fifo_key(g.arrival, g.gid);
            k1 = is_score ? ks : kf;
            k2 = is_score ? kf : ks;
            return ok;
        };
        __syncthreads();
        if (tid == 0) { M->members = 0; M->sec = 0; M->sec_sp = 0.f; M->gexc = 0; M->pn = 0; }
        // ---- rows: exclusive prefix of the row counts (parallel load + block scan)
        const int nrows = IN == MERGE_IN_ROWS ? A.rows.G : A.world;
        for (int r = tid; r < nrows; r += NT) {
            int c = 0;
            if (s < nq)
                c = IN == MERGE_IN_ROWS ? A.rows.cnt[(size_t)s * A.rows.G + r]
                                        : ((const int*)(A.ex_in + (int64_t)r * A.ex_bytes + X.cnt))[s];
            rowoff[r + 1] = c;
        }
        if (tid == 0) rowoff[0] = 0;
        __syncthreads();
        if (tid < 32) {   // one warp scans (nrows <= 1024)
            int carry = 0;
            for (int r0 = 1; r0 <= nrows; r0 += 32) {
                const int r = r0 + lane;
                int v = r <= nrows ? rowoff[r] : 0;
                for (int o = 1; o < 32; o <<= 1) {
                    const int u = __shfl_up_sync(0xffffffffu, v, o);
                    if (lane >= o) v += u;
                }
                if (r <= nrows) rowoff[r] = v + carry;
                carry += __shfl_sync(0xffffffffu, v, 31);
            }
        }
        __syncthreads();
        MDBG(12);
        // ---- members and secondary (rows + this slot's gap requests)
        {
            unsigned long long m = 0;
            u64 sk = 0;
            float ssk = 0.f;
            int gex = 0;
            if (s < nq) {
                for (int r = tid; r < nrows; r += NT) {
                    u64 k;
                    float kp = 0.f;
                    if (IN == MERGE_IN_ROWS) {
                        m += (unsigned long long)A.rows.members[(size_t)s * A.rows.G + r];
                        k = A.rows.sec[(size_t)s * A.rows.G + r];
                    } else {
                        const unsigned char* rec = A.ex_in + (int64_t)r * A.ex_bytes;
                        m += (unsigned long long)((const int64_t*)(rec + X.members))[s];
                        k = ((const u64*)(rec + X.sec))[s];
                        kp = ((const float*)(rec + X.sec_sp))[s];
                    }
                    if (k > sk) { sk = k; ssk = kp; }
                }
            }
            for (long long e = tid; e < ngap_all; e += NT) {
                if (__ldcg(&A.g_slot[e]) != s) continue;
                u64 k1, k2;
                float sp;
                if (gap_keys(gap_entry((uint32_t)e), k1, k2, sp)) {
                    m++;
                    if (k2 > sk) { sk = k2; ssk = sp; }
                } else {
                    gex++;
                }
            }
            for (int o = 16; o; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
            gex = __reduce_add_sync(0xffffffffu, gex);
            const u64 wm = warp_max_u64(sk);
            const unsigned holder = __ballot_sync(0xffffffffu, sk == wm && wm != 0);
            const float wsp = __shfl_sync(0xffffffffu, ssk, holder ? __ffs(holder) - 1 : 0);
            if (lane == 0) {
                if (m) atomicAdd(&M->members, m);
                if (gex) atomicAdd(&M->gexc, gex);
                if (wm) atomicMax(&M->sec, wm);
            }
            __syncthreads();
            if (lane == 0 && wm && wm == M->sec) M->sec_sp = wsp;   // keys are unique: one writer
            __syncthreads();
        }

        MDBG(13);
        // ---- candidate pool: rows entries then this slot's gap requests.  Row keys
        // below the best threshold any CTA published are not in the top-k.
        u64 thr = (IN == MERGE_IN_ROWS && s < nq) ? __ldcg(&A.gthr[s]) : 0ull;
        int pn = 0;
        const int total_rows = rowoff[nrows];
        const long long total = total_rows + ngap_all;
        long long e0 = 0;
        // fast path (rows input, <= 2 keys per lane per row, <= 12 rows per warp): every
        // warp loads all keys of its rows in one go (independent loads in flight), then
        // filters them into the pool; the general loop below then handles only the
        // gap requests of this slot.
        constexpr int kMWarps = NT / 32;
        constexpr int kFR = 12;
        if (IN == MERGE_IN_ROWS && A.rows.cap <= 64 && nrows <= kFR * kMWarps &&
            total_rows <= L.esmem - NT) {
            const int warp_m = tid >> 5;
            u64 kv[kFR][2];
#pragma unroll
            for (int i = 0; i < kFR; i++) {
                const int r = warp_m + i * kMWarps;
                const int c = r < nrows ? rowoff[r + 1] - rowoff[r] : 0;
                const u64* src = A.rows.keys + ((size_t)s * A.rows.G + r) * A.rows.cap;
                kv[i][0] = lane < c ? __ldcg(src + lane) : 0ull;
                kv[i][1] = lane + 32 < c ? __ldcg(src + lane + 32) : 0ull;
            }
            if (tid == 0) M->pn = 0;
            __syncthreads();
#pragma unroll
            for (int i = 0; i < kFR; i++)
#pragma unroll
                for (int h = 0; h < 2; h++)
                    if (kv[i][h] && kv[i][h] >= thr) {
                        const int o = atomicAdd(&M->pn, 1);
                        EWSJF_CHECK(o < L.esmem);
                        uni[o] = kv[i][h];
                    }
            __syncthreads();
            pn = M->pn;
            e0 = total_rows;            // rows done; the loop below appends gap requests only
        }
        while (e0 < total) {
            const int space = L.esmem - pn;
            if (space < NT && pn > kRankMax) {
                pool_shrink<NT>(uni, psp, pn, thr, K, surv, ssp, M);
                continue;
            }
            const int take = (int)(total - e0 < (long long)space ? total - e0 : (long long)space);
            if (tid == 0) M->pn = pn;
            __syncthreads();
            // kU elements per thread per step: their row lookups and loads are issued
            // together (kU loads in flight instead of one L2 round trip each)
            constexpr int kU = 8;
            for (int i0 = tid; i0 < take; i0 += kU * NT) {
                u64 key[kU];
                float sp[kU];
                bool ok[kU];
#pragma unroll
                for (int u = 0; u < kU; u++) {
                    const int i = i0 + u * NT;
                    const long long e = e0 + i;
                    key[u] = 0ull; sp[u] = 0.f; ok[u] = false;
                    if (i < take && e < total_rows) {
                        int lo = 0, hi = nrows;       // row r with rowoff[r] <= e < rowoff[r+1]
                        while (hi - lo > 1) {
                            const int mid = (lo + hi) >> 1;
                            if (rowoff[mid] <= e) lo = mid; else hi = mid;
                        }
                        const int j = (int)(e - rowoff[lo]);
                        if (IN == MERGE_IN_ROWS) {
                            key[u] = __ldcg(&A.rows.keys[((size_t)s * A.rows.G + lo) * A.rows.cap + j]);
                        } else {
                            const unsigned char* rec = A.ex_in + (int64_t)lo * A.ex_bytes;
                            key[u] = ((const u64*)(rec + X.keys))[(size_t)s * K + j];
                            sp[u] = ((const float*)(rec + X.sp))[(size_t)s * K + j];
                        }
                        ok[u] = true;
                    }
                }
#pragma unroll
                for (int u = 0; u < kU; u++) {
                    const int i = i0 + u * NT;
                    const long long e = e0 + i;
                    if (i < take && e >= total_rows && __ldcg(&A.g_slot[e - total_rows]) == s) {
                        u64 k2;
                        ok[u] = gap_keys(gap_entry((uint32_t)(e - total_rows)), key[u], k2, sp[u]);
                    }
                    if (ok[u] && key[u] >= thr) {
                        const int p = atomicAdd(&M->pn, 1);
                        EWSJF_CHECK(p < L.esmem);
                        uni[p] = key[u];
                        if (psp) psp[p] = sp[u];
                    }
                }
            }
            __syncthreads();
            pn = M->pn;
            e0 += take;
        }
        if (pn > kRankMax) pool_shrink<NT>(uni, psp, pn, thr, K, surv, ssp, M);
        MDBG(14);
        // rank sort (keys unique) -> surv[0..pn) descending
        for (int i = tid; i < pn; i += NT) {
            const u64 k = uni[i];
            int r = 0;
            for (int j = 0; j < pn; j++) r += uni[j] > k;
            surv[r] = k;
            if (psp) ssp[r] = psp[i];
        }
        __syncthreads();
        MDBG(15);
        const int nout = pn < K ? pn : K;
        auto payload = [&](int r) -> float {     // s' of ranked entry r
            const u64 k = surv[r];
            if (is_score) return key_sp(k);
            if (IN == MERGE_IN_EXCHANGE) return ssp[r];
            return recompute(key_gid(k));
        };
        const unsigned long long members = M->members;
        const u64 sec = M->sec;
        float sec_payload = 0.f;
        if (sec) {
            if (!is_score) sec_payload = key_sp(sec);                 // SCORE-keyed: s' is the key
            else if (IN == MERGE_IN_EXCHANGE) sec_payload = M->sec_sp;  // carried by the records
            else sec_payload = recompute(key_gid(sec));               // local pool
        }

        if (OUT == MERGE_OUT_FINAL) {
            const int pos = t_pos[s];
            const float qi = (float)(pos + 1);
            for (int r = tid; r < K; r += NT) {
                const size_t o = (size_t)pos * K + r;
                if (r < nout) {
                    A.topk_id[o] = (int64_t)key_gid(surv[r]);
                    A.topk_score[o] = qi * payload(r);
                } else {
                    A.topk_id[o] = -1;
                    A.topk_score[o] = 0.f;
                }
            }
            if (tid == 0) {
                A.count[pos] = (int64_t)members;
                if (members == 0 || nout == 0) {
                    A.head_id[pos] = -1; A.head_score[pos] = 0.f; A.max_score[pos] = 0.f;
                } else if (is_score) {
                    A.head_id[pos] = (int64_t)key_gid(sec);
                    A.head_score[pos] = qi * sec_payload;
                    A.max_score[pos] = qi * key_sp(surv[0]);
                } else {
                    A.head_id[pos] = (int64_t)key_gid(surv[0]);
                    A.head_score[pos] = qi * payload(0);
                    A.max_score[pos] = qi * key_sp(sec);
                }
            }
        } else {   // MERGE_OUT_EXCHANGE: this rank's record
            unsigned char* rec = A.ex_out;
            for (int r = tid; r < nout; r += NT) {
                ((u64*)(rec + X.keys))[(size_t)s * K + r] = surv[r];
                ((float*)(rec + X.sp))[(size_t)s * K + r] = payload(r);
            }
            if (tid == 0) {
                ((int*)(rec + X.cnt))[s] = nout;
                ((int64_t*)(rec + X.members))[s] = (int64_t)members;
                ((u64*)(rec + X.sec))[s] = sec;
                ((float*)(rec + X.sec_sp))[s] = sec_payload;
            }
        }
        if (IN == MERGE_IN_ROWS && s < nq && tid == 0) A.gthr[s] = 0ull;
        if (tid == 0 && M->gexc) atomicAdd(&A.ctr->n_excluded, (unsigned long long)M->gexc);
    }
    if (IN == MERGE_IN_ROWS && OUT == MERGE_OUT_ROUTE)
        for (int i = blockIdx.x * NT + tid; i < nq; i += gridDim.x * NT) A.gthr[i] = 0ull;
    if (OUT == MERGE_OUT_EXCHANGE && blockIdx.x == 0) {   // header + gap entries of this rank
        const int ng = (int)(graw < X.gap_cap ? graw : X.gap_cap);
        for (int i = tid; i < ng; i += NT) ((GapEntry*)(A.ex_out + X.gaps))[i] = A.gap[i];
        if (tid == 0) {
            ExHeader* h = (ExHeader*)(A.ex_out + X.hdr);
            h->gap_count = graw;
            h->n_invalid = (int64_t)__ldcg(&A.ctr->n_invalid);
            h->n_excluded = (int64_t)__ldcg(&A.ctr->n_excluded);
        }
    }

    // ---------------- last CTA: Alg. 1 ArgMax (ties -> lowest index R24), summary, reset
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        const unsigned t = atomicAdd(&A.ctr->ticket, 1u);
        M->is_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!M->is_last || tid >= 32) return;
    __threadfence();
    // Alg. 1 ArgMax over the non-empty queues by head score, ties -> lowest position
    // (one warp: all loads in flight at once, then a warp reduction)
    int primary = -1;
    if (OUT == MERGE_OUT_FINAL) {
        u64 best = 0ull;      // (ordered head score << 32) | ~position, 0 = none
        for (int p = tid; p < nfinal; p += 32) {
            if (__ldcg(&A.count[p]) > 0) {
                const u64 k = ((u64)ord_f32(__ldcg(&A.head_score[p])) << 32) | (u64)(~(u32)p);
                best = k > best ? k : best;
            }
        }
        best = warp_max_u64(best);
        primary = best ? (int)(~(u32)best) : -1;
    }
    if (tid != 0) return;
    long long inv = (long long)__ldcg(&A.ctr->n_invalid) + M->ndrop;
    long long exc = (long long)__ldcg(&A.ctr->n_excluded);
    if (IN == MERGE_IN_EXCHANGE) {
        for (int r = 0; r < A.world; r++) {
            const ExHeader* h = (const ExHeader*)(A.ex_in + (int64_t)r * A.ex_bytes);
            inv += h->n_invalid;
            exc += h->n_excluded;
        }
    }
    if (OUT != MERGE_OUT_EXCHANGE && A.summary) {
        ewsjf_summary sm;
        sm.n_queues = nfinal;
        sm.primary = primary;
        sm.n_invalid = inv;
        sm.n_excluded = exc;
        sm.n_gap = graw;
        sm.n_bubbles = M->nbub;
        sm.n_dropped = M->ndrop;
        sm.status = (gap_overflow || M->ndrop) ? EWSJF_ERR_CAPACITY : ((inv || exc) ? EWSJF_ERR_DOMAIN : EWSJF_OK);
        sm.pad = 0;
        *A.summary = sm;
    }
    A.ctr->n_invalid = 0;
    A.ctr->n_excluded = 0;
    A.ctr->gap_count = 0;
    A.ctr->ticket = 0;
    A.ctr->barrier = 0;
    A.ctr->tiles = 0;
}

}  // namespace ewsjf
