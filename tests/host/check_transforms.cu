// Host-side check of the scheduled 1-D transforms (csrc/transforms.cuh) against the
// matrix form (and the biased forward form), for every variant: random int inputs, exact equality.  Built and run by
// tests/test_transforms_host.py (nvcc, host code only -- no GPU needed).
#include <cstdio>
#include <random>

#include "transforms.cuh"

using namespace sfcb200;

template <int V>
int check(std::mt19937_64& rng) {
    using T = Tab<V>;
    std::uniform_int_distribution<int> d(-200000, 200000);
    int bad = 0;
    for (int trial = 0; trial < 20000; ++trial) {
        long long x[T::n], yf[T::K], yg[T::K], p[T::K], zi[T::M], zg[T::M];
        for (auto& v : x) v = d(rng);
        for (auto& v : p) v = d(rng);
        long long cb[T::K], yb[T::K];
        for (auto& v : cb) v = d(rng);
        fwd1d<V>(x, yf);
        fwd1d_generic<V>(x, yg);
        fwd1d_bias<V>(x, yb, cb);
        for (int k = 0; k < T::K; ++k) bad += yb[k] != yg[k] + cb[k];
        inv1d<V>(p, zi);
        inv1d_generic<V>(p, zg);
        for (int k = 0; k < T::K; ++k) bad += yf[k] != yg[k];
        for (int t = 0; t < T::M; ++t) bad += zi[t] != zg[t];
    }
    std::printf("variant %d: %d mismatches\n", V, bad);
    return bad;
}

int main() {
    std::mt19937_64 rng(1234);
    const int bad = check<0>(rng) + check<1>(rng) + check<2>(rng);
    return bad ? 1 : 0;
}
