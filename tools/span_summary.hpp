// Host side of the whole-grid span trace (ptx.cuh span_mark, -DFIPA_SPAN_TRACE): concurrency,
// mean CTA lifetime split at the epilogue mark, and the implied number of waves.
#pragma once
#include <algorithm>
#include <cstdio>
#include <utility>
#include <vector>

inline void span_summary(const char* name, int nctas) {
    std::vector<unsigned long long> sp(4 * 65536);
    cudaMemcpyFromSymbol(sp.data(), fipa_b200::g_span, sp.size() * sizeof(unsigned long long));
    unsigned long long t_min = ~0ull, t_max = 0;
    double life = 0, epi = 0, body = 0;
    int n = 0, ne = 0;
    std::vector<std::pair<unsigned long long, int>> ev;
    for (int c = 0; c < nctas && c < 65536; ++c) {
        const unsigned long long a0 = sp[4 * c], a1 = sp[4 * c + 1], a2 = sp[4 * c + 2];
        if (!a0 || !a2 || a2 < a0) continue;
        t_min = std::min(t_min, a0);
        t_max = std::max(t_max, a2);
        life += double(a2 - a0);
        if (a1 >= a0 && a1 <= a2) {
            epi += double(a2 - a1);
            body += double(a1 - a0);
            ++ne;
        }
        ev.push_back({a0, 1});
        ev.push_back({a2, -1});
        ++n;
    }
    std::sort(ev.begin(), ev.end());
    int cur = 0, mx = 0;
    for (auto& e : ev) {
        cur += e.second;
        mx = std::max(mx, cur);
    }
    if (n == 0 || mx == 0) {
        printf("%s: no spans recorded\n", name);
        return;
    }
    printf("%s spans: %d CTAs, span %.1f us, max concurrent %d, mean lifetime %.2f us "
           "(start->epilogue %.2f, epilogue %.2f), waves %.2f\n",
           name, n, (t_max - t_min) / 1e3, mx, life / n / 1e3, ne ? body / ne / 1e3 : 0.0, ne ? epi / ne / 1e3 : 0.0,
           double(n) / mx);
}
