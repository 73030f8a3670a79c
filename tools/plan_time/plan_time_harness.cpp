#include "tt_internal.h"
#include <chrono>
#include <cstdio>
#include <vector>
#include <algorithm>
using namespace tt;
namespace tt { int log_level(){return 0;} void log_plan(const Plan&, double, bool){} Plan::~Plan(){} }
int main(int argc, char** argv) {
    FILE* f = fopen("probs.txt", "r");
    std::vector<std::vector<long long>> P;
    int r, e;
    while (fscanf(f, "%d %d", &r, &e) == 2) {
        std::vector<long long> v{r, e};
        for (int i = 0; i < 2 * r; ++i) { long long x; fscanf(f, "%lld", &x); v.push_back(x); }
        P.push_back(v);
    }
    int reps = argc > 1 ? atoi(argv[1]) : 1;
    std::vector<double> ts(P.size() * 0), best(P.size(), 1e30);
    DeviceInfo dev;
    FILE* dump = argc > 2 ? fopen(argv[2], "w") : nullptr;
    for (int rep = 0; rep < reps; ++rep)
    for (size_t pi = 0; pi < P.size(); ++pi) { auto& v = P[pi];
        int rank = v[0], es = v[1];
        int64_t dims[32]; int perm[32];
        for (int i = 0; i < rank; ++i) { dims[i] = v[2 + i]; perm[i] = v[2 + rank + i]; }
        auto t0 = std::chrono::steady_clock::now();
        Plan p; p.rank = rank; p.dims.assign(dims, dims + rank); p.perm.assign(perm, perm + rank);
        p.prob = normalize(rank, dims, perm, es, true);
        int k = widen_factor(p.prob);
        if (k > 1) { Plan nar; nar.prob = p.prob; choose_plan(nar, dev, nullptr, nullptr); p.prob = widen_problem(p.prob, k); }
        choose_plan(p, dev, nullptr, nullptr);
        if (rep == 0 && dump) fprintf(dump, "%s\n", describe_json(p).c_str());
        best[pi] = std::min(best[pi], std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
    }
    std::vector<double> s = best; std::sort(s.begin(), s.end());
    printf("n %zu median %.1f p90 %.1f max %.1f\n", s.size(), s[s.size()/2], s[s.size()*9/10], s.back());
}
