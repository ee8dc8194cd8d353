// Warp-specialised fused backward + optimizer (the UPDATE fast path).
//
// Same semantics as tbe_stream_update_kernel (embedding.py:175-192 aggregate
// in sorted = buffer order, then exactly one optimizer step per touched row,
// embedding.py:212-254), same work split (a task of CHUNK sorted entries owns
// every segment whose head lies in it; rows that run through whole 128-entry
// "hot" chunks fold those chunks' precomputed partials), but the two halves
// of the walk run on different warps:
//
//   producer warp  claims tasks from the atomic work queue, reads the sorted
//                  (key, bag) stream 32 entries at a time (lane-parallel),
//                  and fills shared-memory stages of E entries: each entry's
//                  upstream row, and for each segment head its weight row,
//                  moment and row pointers (cp.async, completion tracked by
//                  the stage's `full` mbarrier);
//   consumer warp  waits on `full`, accumulates the stage's rows in entry
//                  order in registers (one LDS.128 + 4 FADD per entry) and
//                  at each head applies the optimizer to the previous row,
//                  storing straight to HBM; then releases the stage through
//                  its `empty` mbarrier.
//
// Each CTA holds P such pairs with S stages each; one CTA per SM.  The
// producer's per-entry cost is one shuffle + one LDGSTS per 16-byte piece,
// and the consumer never branches on pipeline state per entry, which is what
// made the single-warp walk issue-bound (profiles/r1_backward_variants.md).
#pragma once
// (included inside namespace neo by tbe_backward.cu, after SegParams,
// Window/load_window, the cp.async helpers and hot_chunk_kernel)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
// the barrier's phase also waits for this thread's earlier cp.async copies
__device__ __forceinline__ void mbar_arrive_cp_async(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}
// upper bound on one hardware-suspended wait (the warp wakes as soon as the
// phase completes); the default limit is short and the retry loop then burns
// issue slots that the other role's warps need
#ifndef NEO_PIPE_SUSPEND_NS
#define NEO_PIPE_SUSPEND_NS 1000000
#endif
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity), "r"(NEO_PIPE_SUSPEND_NS)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

#ifndef NEO_PIPE_E
#define NEO_PIPE_E 4
#endif
#ifndef NEO_PIPE_S
#define NEO_PIPE_S 2
#endif
#ifndef NEO_PIPE_CHUNK
#define NEO_PIPE_CHUNK 256
#endif
#ifndef NEO_PIPE_SMEM
#define NEO_PIPE_SMEM (200 * 1024)
#endif
#ifndef NEO_PIPE_MINB
#define NEO_PIPE_MINB 1
#endif
#ifndef NEO_PIPE_MAXP
#define NEO_PIPE_MAXP 16
#endif

constexpr int kHotChunk = 128;  // granularity of hot-chunk partials (hot_chunk_kernel)

template <typename W, typename G, int OPT, int VPL>
struct PipeCfg {
  static constexpr int kVec = 16 / sizeof(W);       // weight elements per 16-byte vector
  static constexpr int kGB = kVec * sizeof(G);      // upstream bytes per lane per vector
  static constexpr int E = NEO_PIPE_E;              // entries per stage
  static constexpr int S = NEO_PIPE_S;              // stages per pair
  static constexpr int kGOff = 0;                   // [E][VPL][32][kGB] upstream rows
  static constexpr int kWOff = kGOff + E * VPL * kWarp * kGB;    // [E][VPL][32][16] weight rows
  static constexpr int kMOff = kWOff + E * VPL * kWarp * 16;     // [E][VPL][32][kVec] f32 moment rows
  static constexpr int kMBytes = OPT == NEO_OPT_ADAGRAD ? E * VPL * kWarp * kVec * 4 : 0;
  static constexpr int kRowMOff = kMOff + kMBytes;               // [E] f32 row-wise moments
  static constexpr int kMetaOff = (kRowMOff + E * 4 + 15) / 16 * 16;
  struct Meta {
    int32_t n;        // entries in this stage
    uint32_t heads;   // bit e: entry e starts a segment
    int32_t flags;    // kFold / kDone
    int32_t pad;
    int64_t cont;     // kFold: first hot chunk the open row continues into
    uint64_t wptr[E];
    uint64_t mptr[E];
    uint64_t key[E];
    int32_t D[E];
  };
  static constexpr int kStage = (kMetaOff + (int)sizeof(Meta) + 127) / 128 * 128;
  static constexpr int P0 = NEO_PIPE_SMEM / (S * kStage);
  static constexpr int P = P0 > NEO_PIPE_MAXP ? NEO_PIPE_MAXP : (P0 < 1 ? 1 : P0);      // producer/consumer pairs per CTA
  // barriers first: an mbarrier that cp.async completions arrive on must sit
  // low in the shared window (at ~200 KB the arrive faulted with an illegal
  // instruction on B200; at offset 0 it does not)
  static constexpr int kBarOff = 0;
  static constexpr int kRingOff = (P * S * 2 * 8 + 127) / 128 * 128;
  static constexpr int kSmem = kRingOff + P * S * kStage;
  static constexpr int kFold = 1, kDone = 2;
};

template <typename W, typename G, typename Key, int OPT, bool FULL, int VPL>
__global__ void __launch_bounds__(2 * PipeCfg<W, G, OPT, VPL>::P * kWarp, NEO_PIPE_MINB)
tbe_pipe_update_kernel(SegParams p, const __grid_constant__ CUtensorMap gmap) {
  using C = PipeCfg<W, G, OPT, VPL>;
  using Meta = typename C::Meta;
  constexpr int kVec = C::kVec, kGB = C::kGB, E = C::E, S = C::S, P = C::P;
  constexpr int CHUNK = NEO_PIPE_CHUNK;
  const unsigned full = 0xffffffffu;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  const int pair = warp % P;
  unsigned char* ring = smem_raw + C::kRingOff + pair * S * C::kStage;
  const uint32_t bars = smem_u32(smem_raw + C::kBarOff) + pair * S * 16;  // full[s] = +16s, empty[s] = +16s+8
  if (threadIdx.x == 0) {
    for (int i = 0; i < P * S; ++i) {
      mbar_init(smem_u32(smem_raw + C::kBarOff) + i * 16, kWarp);  // full: 32 producer lanes
      mbar_init(smem_u32(smem_raw + C::kBarOff) + i * 16 + 8, 1);   // empty: consumer lane 0
    }
  }
  __syncthreads();
  const Key* keys = reinterpret_cast<const Key*>(p.keys);
  const int64_t N = p.N;
  // No L2::cache_hint on the producer's copies: with P >= 2 pairs and S >= 2
  // stages, hinted cp.async (createpolicy evict_last) in this kernel raised
  // "illegal instruction" on B200 wherever the policy was created; unhinted
  // copies are bitwise-identical in result and were not slower.

  if (warp >= P) {
    // ------------------------------------------------------------ producer
    const G* gbase = reinterpret_cast<const G*>(p.grad);
    const int64_t ntasks = (N + CHUNK - 1) / CHUNK;
    unsigned long long* counter = reinterpret_cast<unsigned long long*>(p.chunk_counter);
    int s = 0;
    uint32_t ephase = 1;  // stages start empty
    auto acquire = [&]() -> unsigned char* {
      mbar_wait(bars + s * 16 + 8, ephase);
      return ring + s * C::kStage;
    };
    auto publish = [&]() {
      mbar_arrive_cp_async(bars + s * 16);
      mbar_arrive(bars + s * 16);
      if (++s == S) {
        s = 0;
        ephase ^= 1;
      }
    };
    // emit entries [l, l+n) of window w into one stage
    auto emit = [&](const Window& w, int l, int n) {
      unsigned char* st = acquire();
      Meta& m = *reinterpret_cast<Meta*>(st + C::kMetaOff);
      const unsigned hm = (w.heads >> l) & (n == 32 ? full : ((1u << n) - 1u));
      const int e_l = lane - l;
      if (e_l >= 0 && e_l < n && ((hm >> e_l) & 1u)) {
        m.wptr[e_l] = w.wptr;
        m.mptr[e_l] = w.mptr;
        m.key[e_l] = w.key;
        m.D[e_l] = w.D;
      }
      if (lane == 0) {
        m.n = n;
        m.heads = hm;
        m.flags = 0;
      }
      unsigned char* gs = st + C::kGOff;
      bool staged = false;
      if (FULL && p.tma) {
        // one gather4 stages the stage's rows when they come from one table
        const int32_t my_t = (lane >= l && lane < l + n) ? w.tt : -1;
        const int32_t t0 = __shfl_sync(full, w.tt, l);
        if (n == E && E == 4 && __all_sync(full, my_t == -1 || my_t == t0)) {
          const int32_t dcol0 = __shfl_sync(full, w.dcol, l);
          uint32_t r[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) r[q] = (uint32_t)__shfl_sync(full, w.grow, l + q);
          if (lane == 0) {
            // expect the bytes before the copy is issued; the plain arrive in publish() follows
            asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(bars + s * 16),
                         "r"(4u * (uint32_t)(kWarp * kGB * VPL))
                         : "memory");
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                "%3, %4, %5, %6}], [%7];\n" ::"r"(smem_u32(gs)),
                "l"(&gmap), "r"(dcol0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(bars + s * 16)
                : "memory");
          }
          staged = true;
        }
      }
#pragma unroll 4
      for (int e = 0; e < (staged ? 0 : n); ++e) {
        const G* grow = gbase + __shfl_sync(full, w.gofs, l + e);
        int De = 0;
        if (!FULL) De = __shfl_sync(full, w.D, l + e);
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          if (FULL || (lane + v * kWarp) * kVec < De) {
            const G* src = grow + (lane + v * kWarp) * kVec;
            unsigned char* dst = gs + ((e * VPL + v) * kWarp + lane) * kGB;
#pragma unroll
            for (int b = 0; b < kGB; b += 16)
              cp_async(dst + b, reinterpret_cast<const char*>(src) + b, kGB < 16 ? kGB : 16);
          }
        }
      }
      unsigned h = hm;
      while (h) {
        const int e = __ffs(h) - 1;
        h &= h - 1;
        const W* wrow = reinterpret_cast<const W*>(__shfl_sync(full, w.wptr, l + e));
        int De = 0;
        if (!FULL) De = __shfl_sync(full, w.D, l + e);
        if (OPT != NEO_OPT_NONE) {  // DENSE mode (OPT_NONE) only writes the row
#pragma unroll
          for (int v = 0; v < VPL; ++v)
            if (FULL || (lane + v * kWarp) * kVec < De)
              cp_async(st + C::kWOff + ((e * VPL + v) * kWarp + lane) * 16, wrow + (lane + v * kWarp) * kVec, 16);
        }
        if (OPT == NEO_OPT_ROWWISE_ADAGRAD) {
          const uint64_t mp = __shfl_sync(full, w.mptr, l + e);
          if (lane == 0) cp_async(st + C::kRowMOff + e * 4, reinterpret_cast<const float*>(mp), 4);
        } else if (OPT == NEO_OPT_ADAGRAD) {
          const float* mrow = reinterpret_cast<const float*>(__shfl_sync(full, w.mptr, l + e));
#pragma unroll
          for (int v = 0; v < VPL; ++v)
            if (FULL || (lane + v * kWarp) * kVec < De) {
#pragma unroll
              for (int b = 0; b < kVec * 4; b += 16)
                cp_async(st + C::kMOff + ((e * VPL + v) * kWarp + lane) * kVec * 4 + b,
                         reinterpret_cast<const char*>(mrow + (lane + v * kWarp) * kVec) + b, 16);
            }
        }
      }
      publish();
    };
    auto emit_flag = [&](int flags, int64_t cont) {
      unsigned char* st = acquire();
      Meta& m = *reinterpret_cast<Meta*>(st + C::kMetaOff);
      if (lane == 0) {
        m.n = 0;
        m.heads = 0;
        m.flags = flags;
        m.cont = cont;
      }
      publish();
    };

    unsigned long long claim = 0;
    if (lane == 0) claim = atomicAdd(counter, 1ull);
    for (;;) {
      const int64_t task = (int64_t)__shfl_sync(full, claim, 0);
      if (task >= ntasks) break;
      if (lane == 0) claim = atomicAdd(counter, 1ull);  // next claim in flight
      const int64_t c0 = task * CHUNK;
      const int64_t cend = c0 + CHUNK;
      Window w;
      uint64_t prev = c0 > 0 ? (uint64_t)keys[c0 - 1] : ~0ull;
      int l = -1;
      for (int64_t wb = c0; wb < cend && wb < N; wb += kWarp) {
        load_window<W, G, Key, OPT>(p, wb, prev, lane, w);
        if (w.heads) {
          l = __ffs(w.heads) - 1;
          break;
        }
        prev = __shfl_sync(full, w.key, kWarp - 1);
      }
      if (l < 0 || !((w.live >> l) & 1u)) continue;
      for (;;) {
        // the range ends at the first head at or after cend, or the first invalid entry
        const int64_t pos = w.base + lane;
        const unsigned beyond = __ballot_sync(full, pos >= cend);
        const unsigned term = ((w.heads & beyond) | ~w.live) & (full << l);
        const int lend = term ? __ffs(term) - 1 : kWarp;
        while (l < lend) {
          const int n = lend - l < E ? lend - l : E;
          emit(w, l, n);
          l += n;
        }
        if (term) break;
        const int64_t nb = w.base + kWarp;
        if (nb >= N) break;
        if (nb % kHotChunk == 0 && p.chunk_slot[nb / kHotChunk] >= 0) {
          emit_flag(C::kFold, nb / kHotChunk);  // the open row runs through hot chunks
          break;
        }
        const uint64_t last = __shfl_sync(full, w.key, kWarp - 1);
        load_window<W, G, Key, OPT>(p, nb, last, lane, w);
        l = 0;
      }
    }
    emit_flag(C::kDone, -1);
    cp_wait<0>();  // no thread may exit with copies into shared memory in flight
    return;
  }

  // -------------------------------------------------------------- consumer
  const float lr = (float)p.lr, eps = (float)p.eps;
  float acc[VPL * kVec];
#pragma unroll
  for (int e = 0; e < VPL * kVec; ++e) acc[e] = 0.f;
  uint4 wr[VPL];          // staged weight row of the open segment (raw W)
  float mw[OPT == NEO_OPT_ADAGRAD ? VPL * kVec : 1];  // its element-wise moments
  float mrow = 0.f;
  uint64_t cw = 0, cm = 0, ckey = 0;
  int cD = FULL ? kWarp * kVec * VPL : 0;
  bool open = false;

  auto live_at = [&](int v) -> bool { return FULL || (lane + v * kWarp) * kVec < cD; };

  auto finalize = [&]() {  // exactly one optimizer step for the open row
    if (OPT == NEO_OPT_NONE) {  // DENSE mode: the aggregated gradient row itself
      float* drow = reinterpret_cast<float*>(cw);
#pragma unroll
      for (int v = 0; v < VPL; ++v)
        if (live_at(v))
#pragma unroll
          for (int e = 0; e < kVec; e += 4)
            *reinterpret_cast<float4*>(drow + (lane + v * kWarp) * kVec + e) =
                make_float4(acc[v * kVec + e], acc[v * kVec + e + 1], acc[v * kVec + e + 2], acc[v * kVec + e + 3]);
#pragma unroll
      for (int e = 0; e < VPL * kVec; ++e) acc[e] = 0.f;
      return;
    }
    if (!FULL) {
#pragma unroll
      for (int v = 0; v < VPL; ++v)
        if (!live_at(v))
#pragma unroll
          for (int e = 0; e < kVec; ++e) acc[v * kVec + e] = 0.f;
    }
    float ss = 0.f;
    bool live_row = true;
    if (OPT == NEO_OPT_ROWWISE_ADAGRAD) {
#pragma unroll
      for (int e = 0; e < VPL * kVec; ++e) ss += acc[e] * acc[e];
      ss = warp_sum(ss);
    }
    if (OPT == NEO_OPT_ADAGRAD || (OPT == NEO_OPT_ROWWISE_ADAGRAD && ss == 0.f)) {
      // an identically zero gradient leaves the row untouched (embedding.py:223);
      // ss can also underflow to 0 for tiny nonzero gradients, so vote
      bool nz = false;
#pragma unroll
      for (int e = 0; e < VPL * kVec; ++e) nz |= acc[e] != 0.f;
      live_row = __any_sync(full, nz);
    }
    if (live_row) {
      float scale = lr;
      if (OPT == NEO_OPT_ROWWISE_ADAGRAD) {
        const float invD = FULL ? 1.0f / (float)(kWarp * kVec * VPL) : __frcp_rn((float)cD);
        const float m = mrow + ss * invD;
        if (lane == 0) *reinterpret_cast<float*>(cm) = m;
        scale = __fdividef(lr, __fsqrt_rn(m) + eps);
      }
      W* wrow = reinterpret_cast<W*>(cw);
      float* mrowp = reinterpret_cast<float*>(cm);
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        if (!live_at(v)) continue;
        const W* wv = reinterpret_cast<const W*>(&wr[v]);
        Vec<W, kVec> o;
        float mo[kVec];
#pragma unroll
        for (int e = 0; e < kVec; ++e) {
          const float w = Elem<W>::to_f(wv[e]);
          const float a = acc[v * kVec + e];
          if (OPT == NEO_OPT_ADAGRAD) {
            const float mj = mw[v * kVec + e] + a * a;
            mo[e] = mj;
            o.v[e] = Elem<W>::from_f(w - __fdividef(lr * a, __fsqrt_rn(mj) + eps));
          } else {
            o.v[e] = Elem<W>::from_f(w - a * scale);
          }
        }
        *reinterpret_cast<uint4*>(wrow + (lane + v * kWarp) * kVec) = *reinterpret_cast<const uint4*>(&o);
        if (OPT == NEO_OPT_ADAGRAD) {
#pragma unroll
          for (int e = 0; e < kVec; e += 4)
            *reinterpret_cast<float4*>(mrowp + (lane + v * kWarp) * kVec + e) =
                make_float4(mo[e], mo[e + 1], mo[e + 2], mo[e + 3]);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < VPL * kVec; ++e) acc[e] = 0.f;
  };

  auto fold = [&](int64_t c) {  // hot-chunk partials in chunk order, then the row's tail
    const int64_t nhot = (N + kHotChunk - 1) / kHotChunk;
    for (; c < nhot; ++c) {
      const int32_t slot = p.chunk_slot[c];
      if (slot < 0) break;
      const float* src = p.pool + (int64_t)slot * p.max_dim;
#pragma unroll
      for (int v = 0; v < VPL; ++v)
        if (live_at(v))
#pragma unroll
          for (int e = 0; e < kVec; ++e) acc[v * kVec + e] += src[(lane + v * kWarp) * kVec + e];
    }
    const G* gbase = reinterpret_cast<const G*>(p.grad);
    for (int64_t j = c * kHotChunk; j < N; ++j) {
      if ((uint64_t)keys[j] != ckey) break;
      const int32_t bag = p.bags[j];
      const int32_t t = bag / (int32_t)p.B;
      const G* src = gbase + ((int64_t)bag - (int64_t)t * p.B) * p.grad_stride + p.dim_offsets[t];
#pragma unroll
      for (int v = 0; v < VPL; ++v)
        if (live_at(v))
#pragma unroll
          for (int e = 0; e < kVec; ++e) acc[v * kVec + e] += Elem<G>::to_f(src[(lane + v * kWarp) * kVec + e]);
    }
  };

  int s = 0;
  uint32_t fphase = 0;
  for (;;) {
    mbar_wait(bars + s * 16, fphase);
    const unsigned char* st = ring + s * C::kStage;
    const Meta& m = *reinterpret_cast<const Meta*>(st + C::kMetaOff);
    const int n = m.n;
    const unsigned heads = m.heads;
    const int flags = m.flags;
    if (flags & C::kDone) break;
    if (flags & C::kFold) {
      fold(m.cont);
      finalize();
      open = false;
    } else {
      // all of the stage's upstream rows up front: E independent LDS in flight
      constexpr int kW8 = kGB / 8;  // 8-byte words per lane per vector
      uint2 gv[E][VPL][kW8];
#pragma unroll
      for (int e = 0; e < E; ++e)
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          const unsigned char* src = st + C::kGOff + ((e * VPL + v) * kWarp + lane) * kGB;
          if (e < n) {
            if constexpr (kW8 % 2 == 0) {
#pragma unroll
              for (int b = 0; b < kW8; b += 2) {
                const uint4 x = *reinterpret_cast<const uint4*>(src + b * 8);
                gv[e][v][b] = make_uint2(x.x, x.y);
                gv[e][v][b + 1] = make_uint2(x.z, x.w);
              }
            } else {
              gv[e][v][0] = *reinterpret_cast<const uint2*>(src);
            }
          } else {
#pragma unroll
            for (int b = 0; b < kW8; ++b) gv[e][v][b] = make_uint2(0, 0);
          }
        }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if (e < n) {
          if ((heads >> e) & 1u) {
            if (open) finalize();
            open = true;
            if (OPT != NEO_OPT_NONE) {
#pragma unroll
              for (int v = 0; v < VPL; ++v)
                wr[v] = *reinterpret_cast<const uint4*>(st + C::kWOff + ((e * VPL + v) * kWarp + lane) * 16);
            }
            if (OPT == NEO_OPT_ROWWISE_ADAGRAD) mrow = *reinterpret_cast<const float*>(st + C::kRowMOff + e * 4);
            if (OPT == NEO_OPT_ADAGRAD) {
#pragma unroll
              for (int v = 0; v < VPL; ++v)
#pragma unroll
                for (int q = 0; q < kVec; ++q)
                  mw[v * kVec + q] = reinterpret_cast<const float*>(
                      st + C::kMOff + ((e * VPL + v) * kWarp + lane) * kVec * 4)[q];
            }
            cw = m.wptr[e];
            cm = m.mptr[e];
            ckey = m.key[e];
            if (!FULL) cD = m.D[e];
          }
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            const G* gq = reinterpret_cast<const G*>(&gv[e][v][0]);
#pragma unroll
            for (int q = 0; q < kVec; ++q) acc[v * kVec + q] += Elem<G>::to_f(gq[q]);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(bars + s * 16 + 8);
    if (++s == S) {
      s = 0;
      fphase ^= 1;
    }
  }
  if (open) finalize();
}

