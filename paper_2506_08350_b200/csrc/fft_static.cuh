// Compile-time-planned Stockham FFT over a batch held in shared memory (sm_100a).
//
// The radices, the transform length N, the batch width NB and the thread count NT
// are template parameters, so every stage is fully unrolled: butterfly indices,
// j % ns and the twiddle strides fold to constants and each codelet is
// instantiated only where it is used (the runtime-planned engine in fft.cuh
// must keep every codelet live and spends 255 registers per thread).
//
// Data flow of one transform batch:
//   stage 0 reads through a caller functor (straight from HBM: no staging copy),
//   stages 1..S-1 read shared memory,
//   stages 0..S-2 write shared memory (in place: every thread first loads all
//   of its butterflies into registers, then a barrier, then writes),
//   stage S-1 writes through a caller functor (fused epilogue: scale, |.|^2,
//   transfer-function products, spectrum accumulation...).
// The functors receive (q, r, b, i[, v]): q = butterfly slot of this thread,
// r = element within the butterfly (both compile-time after unrolling, so
// per-thread register arrays can be indexed by them), b = transform in the
// batch, i = element index.  The last stage of a forward plan [R1..Rk] and the
// first stage of the reversed inverse plan [Rk..R1] touch the same (q, r, b, i)
// per thread, which lets a spectrum stay in registers between them.
//
// Shared-memory layout (PadLayout): element i of transform b at
// [(i + (i / R1) * pad) * NB + b], R1 = the plan's first radix (batch index
// fastest; a warp touches 32 / NB consecutive rows of NB complex values).
// Every index a stage forms is a butterfly base plus a compile-time multiple of
// R1 (or, in the first stage, R1 j + r with r < R1), so each shared-memory access
// is one base register plus an immediate offset; pad is the smallest that
// spreads the first stage's stride-R1 writes evenly over the banks.
#pragma once

#include "fft.cuh"

namespace holo_cuda {

template <int... Rs>
struct Radices {};

template <class P>
struct RevPlan;
template <>
struct RevPlan<Radices<>> {
    using type = Radices<>;
};
template <int R, int... Rs>
struct RevPlan<Radices<R, Rs...>> {
    template <class A, int X>
    struct Append;
    template <int... As, int X>
    struct Append<Radices<As...>, X> {
        using type = Radices<As..., X>;
    };
    using type = typename Append<typename RevPlan<Radices<Rs...>>::type, R>::type;
};

template <int N, int NB, int NT>
struct Batch {
    static constexpr int kN = N, kNB = NB, kNT = NT;
};

template <class P>
struct FirstRadix;
template <int R, int... Rs>
struct FirstRadix<Radices<R, Rs...>> {
    static constexpr int value = R;
};

// smallest pad for which one warp's first-stage writes (lanes b = t % NB,
// j = t / NB, element R1 j, 8-byte complex = two 4-byte banks) hit no bank more
// than the two times a 256-byte access needs anyway
constexpr int pick_pad(int R1, int NB) {
    for (int p = 0; p < 64; ++p) {
        int cnt[32] = {};
        int worst = 0;
        for (int t = 0; t < 32; ++t) {
            const int b = t % NB, j = t / NB;
            const int word = 2 * ((R1 + p) * j * NB + b);
            for (int k = 0; k < 2; ++k) {
                const int c = ++cnt[(word + k) % 32];
                worst = c > worst ? c : worst;
            }
        }
        if (worst <= 2) return p;
    }
    return 0;
}

template <int N, int NB, int R1>
struct PadLayout {
    static constexpr int kPad = pick_pad(R1, NB);
    static constexpr int kElems = (NB * (N + (N / R1) * kPad) + 1) & ~1;  // even: 16-byte multiple
    static constexpr int kR1 = R1;
    static __device__ __forceinline__ int at(int b, int i) { return (i + (i / R1) * kPad) * NB + b; }
    // at(b, i + d) - at(b, i) for d a multiple of R1
    static constexpr int off(int d) { return (d + (d / R1) * kPad) * NB; }
};

// shared-memory elements of batch B for plan P and its reverse (the inverse)
template <class B, class P>
struct FftSmem {
    static constexpr int kF = PadLayout<B::kN, B::kNB, FirstRadix<P>::value>::kElems;
    static constexpr int kI = PadLayout<B::kN, B::kNB, FirstRadix<typename RevPlan<P>::type>::value>::kElems;
    static constexpr int kElems = kF > kI ? kF : kI;
};

// One stage: radix R, ns = product of the earlier radices; FIRST/LAST select the
// functor paths.
template <class T, int DIR, class B, class Lay, int R, int NS, bool FIRST, bool LAST>
struct Stage {
    static constexpr int N = B::kN, NB = B::kNB, NT = B::kNT;
    static constexpr int M = N / R;
    static constexpr int TOT = M * NB;
    static constexpr int BPT = (TOT + NT - 1) / NT;

    // Twiddles w^r, r < R: w is read from the table (consecutive k: no bank
    // conflicts), the powers of two squared up from it and the others formed as
    // products of them (w^r = w^p w^(r-p), p the largest power of two below r) --
    // FMA-pipe work instead of shared-memory reads (the row pass's bottleneck),
    // at most 6 fp32 roundings.
    static __device__ __forceinline__ void butterfly(cx<T>* v, int j, const cx<T>* __restrict__ tw) {
        const int k = j % NS;
        if constexpr (NS > 1) {
            const int step = (N / (NS * R)) * k;
            cx<T> w[R];
#pragma unroll
            for (int r = 1; r < R; ++r) {
                if (r == 1) {
                    w[1] = tw[step];
                    if (DIR > 0) w[1].y = -w[1].y;
                } else if ((r & (r - 1)) == 0) {
                    w[r] = w[r / 2] * w[r / 2];
                } else {
                    const int p = 1 << (31 - __clz(r));
                    w[r] = w[p] * w[r - p];
                }
                v[r] = v[r] * w[r];
            }
        }
        Dft<R, DIR, T>::run(v);
    }

    template <class Load, class Store, class Hook>
    static __device__ __forceinline__ void run(cx<T>* sm, const cx<T>* __restrict__ tw, Load& load, Store& store,
                                               Hook& hook) {
        if constexpr (FIRST || LAST) {
            // Streaming stage: it either only writes sm (first) or only reads it
            // (last), so butterflies go one by one with R live values each.
#pragma unroll
            for (int q = 0; q < BPT; ++q) {
                const int t = threadIdx.x + q * NT;
                if (TOT % NT == 0 || t < TOT) {
                    const int b = t % NB, j = t / NB;
                    cx<T> v[R];
                    if constexpr (!FIRST) {
                        static_assert(M % Lay::kR1 == 0, "stage reads must step by multiples of R1");
                    }
                    const int a0 = FIRST ? 0 : Lay::at(b, j);
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int i = j + r * M;
                        if constexpr (FIRST)
                            v[r] = load(q, r, b, i);
                        else
                            v[r] = sm[a0 + Lay::off(r * M)];
                    }
                    butterfly(v, j, tw);
                    const int k = j % NS;
                    const int base = (j - k) * R + k;
                    if constexpr (!LAST) {
                        static_assert(NS == 1 && R == Lay::kR1, "a streaming write stage is the plan's first");
                    }
                    const int aw = LAST ? 0 : Lay::at(b, base);
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int i = base + r * NS;
                        if constexpr (LAST)
                            store(q, r, b, i, v[r]);
                        else
                            sm[aw + r * NB] = v[r];  // base = R1 j, r < R1
                    }
                }
            }
            // first: writes visible to the next stage; last: every sm read done
            // before the caller (or its next transform) writes sm again
            if constexpr (!(FIRST && LAST)) __syncthreads();
            if constexpr (FIRST) hook();  // every load of the first stage has completed
        } else {
            run_middle(sm, tw);
        }
    }

    // Middle stage, in place: hold all of this thread's butterflies, barrier, write.
    static __device__ __forceinline__ void run_middle(cx<T>* sm, const cx<T>* __restrict__ tw) {
        cx<T> v[BPT][R];
#pragma unroll
        for (int q = 0; q < BPT; ++q) {
            const int t = threadIdx.x + q * NT;
            if (TOT % NT == 0 || t < TOT) {
                const int b = t % NB, j = t / NB;
                static_assert(M % Lay::kR1 == 0 && NS % Lay::kR1 == 0, "middle stages step by multiples of R1");
                const int a0 = Lay::at(b, j);
#pragma unroll
                for (int r = 0; r < R; ++r) v[q][r] = sm[a0 + Lay::off(r * M)];
            }
        }
        __syncthreads();  // every read of sm done before any write
#pragma unroll
        for (int q = 0; q < BPT; ++q) {
            const int t = threadIdx.x + q * NT;
            if (TOT % NT == 0 || t < TOT) {
                const int b = t % NB, j = t / NB;
                butterfly(v[q], j, tw);
                const int k = j % NS;
                const int base = (j - k) * R + k;
                const int aw = Lay::at(b, base);
#pragma unroll
                for (int r = 0; r < R; ++r) sm[aw + Lay::off(r * NS)] = v[q][r];
            }
        }
        __syncthreads();
    }
};

template <class T, int DIR, class B, class Lay, int NS, bool FIRST, class P>
struct Stages;

template <class T, int DIR, class B, class Lay, int NS, bool FIRST, int R>
struct Stages<T, DIR, B, Lay, NS, FIRST, Radices<R>> {
    template <class Load, class Store, class Hook>
    static __device__ __forceinline__ void run(cx<T>* sm, const cx<T>* tw, Load& load, Store& store, Hook& hook) {
        Stage<T, DIR, B, Lay, R, NS, FIRST, true>::run(sm, tw, load, store, hook);
    }
};

template <class T, int DIR, class B, class Lay, int NS, bool FIRST, int R, int R2, int... Rs>
struct Stages<T, DIR, B, Lay, NS, FIRST, Radices<R, R2, Rs...>> {
    template <class Load, class Store, class Hook>
    static __device__ __forceinline__ void run(cx<T>* sm, const cx<T>* tw, Load& load, Store& store, Hook& hook) {
        Stage<T, DIR, B, Lay, R, NS, FIRST, false>::run(sm, tw, load, store, hook);
        Stages<T, DIR, B, Lay, NS * R, false, Radices<R2, Rs...>>::run(sm, tw, load, store, hook);
    }
};

// Transform a batch: load(q, r, b, i) feeds stage 0, store(q, r, b, i, v) takes the result.
// The caller must separate two consecutive calls that share sm by a barrier only if
// it touches sm itself in between (the last stage ends its sm reads with a barrier).
// hook() runs once every thread has finished the first stage's loads (after its
// barrier; plans of two or more stages), e.g. to refill the load source.
template <class T, int DIR, class B, class P, class Load, class Store, class Hook>
__device__ __forceinline__ void fft_static(cx<T>* sm, const cx<T>* __restrict__ tw, Load load, Store store,
                                           Hook hook) {
    using Lay = PadLayout<B::kN, B::kNB, FirstRadix<P>::value>;
    Stages<T, DIR, B, Lay, 1, true, P>::run(sm, tw, load, store, hook);
}
template <class T, int DIR, class B, class P, class Load, class Store>
__device__ __forceinline__ void fft_static(cx<T>* sm, const cx<T>* __restrict__ tw, Load load, Store store) {
    fft_static<T, DIR, B, P>(sm, tw, load, store, [] {});
}

// Asynchronous 16-byte global -> shared copies (LDGSTS), grouped by commit.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Last-stage geometry of plan P (for register arrays living across transforms).
template <class B, class P>
struct LastStage;
template <class B, int R>
struct LastStage<B, Radices<R>> {
    static constexpr int kR = R;
    static constexpr int kBPT = ((B::kN / R) * B::kNB + B::kNT - 1) / B::kNT;
};
template <class B, int R, int R2, int... Rs>
struct LastStage<B, Radices<R, R2, Rs...>> : LastStage<B, Radices<R2, Rs...>> {};

}  // namespace holo_cuda
