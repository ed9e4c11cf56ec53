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
// Shared-memory layout: element i of transform b at [i * NB + b] (batch index
// fastest); a warp then touches 32 / NB consecutive rows of NB complex values.
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
    // one pad slot per 32 complex values: the stride-R writes of early Stockham
    // stages (i = R j + r) would otherwise land 32 lanes on one bank pair
    static constexpr int kSmemElems = ((N * NB + (N * NB) / 32 + 1) + 1) & ~1;  // even: 16-byte multiple
    static __device__ __forceinline__ int at(int b, int i) {
        const int c = i * NB + b;
        return c + (c >> 5);
    }
};

// One stage: radix R, ns = product of the earlier radices; FIRST/LAST select the
// functor paths.
template <class T, int DIR, class B, int R, int NS, bool FIRST, bool LAST>
struct Stage {
    static constexpr int N = B::kN, NB = B::kNB, NT = B::kNT;
    static constexpr int M = N / R;
    static constexpr int TOT = M * NB;
    static constexpr int BPT = (TOT + NT - 1) / NT;

    static __device__ __forceinline__ void butterfly(cx<T>* v, int j, const cx<T>* __restrict__ tw) {
        const int k = j % NS;
        if constexpr (NS > 1) {
            const int step = (N / (NS * R)) * k;
#pragma unroll
            for (int r = 1; r < R; ++r) {
                cx<T> w = tw[r * step];
                if (DIR > 0) w.y = -w.y;
                v[r] = v[r] * w;
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
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int i = j + r * M;
                        if constexpr (FIRST)
                            v[r] = load(q, r, b, i);
                        else
                            v[r] = sm[B::at(b, i)];
                    }
                    butterfly(v, j, tw);
                    const int k = j % NS;
                    const int base = (j - k) * R + k;
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int i = base + r * NS;
                        if constexpr (LAST)
                            store(q, r, b, i, v[r]);
                        else
                            sm[B::at(b, i)] = v[r];
                    }
                }
            }
            // first: writes visible to the next stage; last: every sm read done
            // before the caller (or its next transform) writes sm again
            if constexpr (!(FIRST && LAST)) __syncthreads();
            if constexpr (FIRST) hook();  // every load of the first stage has completed
            return;
        }
        // Middle stage, in place: hold all of this thread's butterflies, barrier, write.
        cx<T> v[BPT][R];
#pragma unroll
        for (int q = 0; q < BPT; ++q) {
            const int t = threadIdx.x + q * NT;
            if (TOT % NT == 0 || t < TOT) {
                const int b = t % NB, j = t / NB;
#pragma unroll
                for (int r = 0; r < R; ++r) v[q][r] = sm[B::at(b, j + r * M)];
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
#pragma unroll
                for (int r = 0; r < R; ++r) sm[B::at(b, base + r * NS)] = v[q][r];
            }
        }
        __syncthreads();
    }
};

template <class T, int DIR, class B, int NS, bool FIRST, class P>
struct Stages;

template <class T, int DIR, class B, int NS, bool FIRST, int R>
struct Stages<T, DIR, B, NS, FIRST, Radices<R>> {
    template <class Load, class Store, class Hook>
    static __device__ __forceinline__ void run(cx<T>* sm, const cx<T>* tw, Load& load, Store& store, Hook& hook) {
        Stage<T, DIR, B, R, NS, FIRST, true>::run(sm, tw, load, store, hook);
    }
};

template <class T, int DIR, class B, int NS, bool FIRST, int R, int R2, int... Rs>
struct Stages<T, DIR, B, NS, FIRST, Radices<R, R2, Rs...>> {
    template <class Load, class Store, class Hook>
    static __device__ __forceinline__ void run(cx<T>* sm, const cx<T>* tw, Load& load, Store& store, Hook& hook) {
        Stage<T, DIR, B, R, NS, FIRST, false>::run(sm, tw, load, store, hook);
        Stages<T, DIR, B, NS * R, false, Radices<R2, Rs...>>::run(sm, tw, load, store, hook);
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
    Stages<T, DIR, B, 1, true, P>::run(sm, tw, load, store, hook);
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
