// Host sanitizer driver (ASan + UBSan): the planner (normalise, widen,
// classify, tile search, slot-dim and vector-gather layouts, describe) on
// the suite shapes and on seeded random problems with random options, fully
// on the host (offline plans, no CUDA runtime calls).
//   g++ -fsanitize=address,undefined -g -O1 planner_fuzz.cpp planner.cpp
#include "../../paper_1705_01598_b200/csrc/tt_internal.h"

#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

using namespace tt;
namespace tt {
Plan::~Plan() { delete narrow; }
void destroy_shard(ShardInfo*) {}
int shard_launches(const ShardInfo*) { return 0; }
std::string describe_shard_json(const Plan&) { return ""; }
}  // namespace tt

static int plan_one(const std::vector<int64_t>& d, const std::vector<int>& p, int E,
                    const tt_plan_options_t* o, bool strided, std::mt19937_64& rng) {
    const int n = (int)d.size();
    if (validate(n, d.data(), p.data(), E) != TT_SUCCESS) return 0;
    DeviceInfo dev;
    Plan pl;
    pl.rank = n;
    pl.dims = d;
    pl.perm = p;
    if (strided) {
        std::vector<int64_t> si(n), so(n);
        int64_t acc = 1;
        for (int i = 0; i < n; ++i) { si[i] = acc; acc *= d[i] + (rng() % 3); }
        acc = 1;
        for (int j = 0; j < n; ++j) { so[j] = acc; acc *= d[p[j]] + (rng() % 2); }
        pl.prob = normalize_strided(n, d.data(), p.data(), E, si.data(), so.data(), true);
    } else {
        pl.prob = normalize(n, d.data(), p.data(), E, !(o && o->no_fusion));
        const int k = (o && o->no_widen) ? 1 : widen_factor(pl.prob);
        if (k > 1) pl.prob = widen_problem(pl.prob, k);
    }
    const tt_status_t st = choose_plan(pl, dev, o, nullptr);
    if (st == TT_SUCCESS) {
        const std::string j = describe_json(pl);
        if (j.size() < 10) return 1;
    }
    return 0;
}

int main() {
    std::mt19937_64 rng(1705);
    int bad = 0, plans = 0;
    for (int it = 0; it < 3000; ++it) {
        const int n = 1 + (int)(rng() % 12);
        std::vector<int64_t> d(n);
        double vol = 1;
        for (auto& x : d) {
            x = 1 + (int64_t)(rng() % (n <= 3 ? 3000 : n <= 6 ? 60 : 9));
            vol *= (double)x;
        }
        if (vol > 4e8) continue;
        std::vector<int> p(n);
        for (int i = 0; i < n; ++i) p[i] = i;
        std::shuffle(p.begin(), p.end(), rng);
        const int E = (rng() & 1) ? 4 : 8;
        tt_plan_options_t o{};
        const int mode = (int)(rng() % 6);
        if (mode == 1) o.vector_gather = 1, o.stages = 3 + (int)(rng() % 2);
        if (mode == 2) o.slot_dims = 1, o.stages = (rng() & 1) ? 4 : 0;
        if (mode == 3) o.kernel = TT_KERNEL_TILE, o.run_in = 1 << (rng() % 9), o.run_out = 1 << (rng() % 9);
        if (mode == 4) o.accumulate = 1;
        bad += plan_one(d, p, E, mode ? &o : nullptr, mode == 5, rng);
        ++plans;
    }
    std::printf("planner fuzz: %d plans, %d bad descriptions\n", plans, bad);
    return bad != 0;
}
