#include "tt_internal.h"
#include <cstdio>
#include <vector>
using namespace tt;
namespace tt { int log_level(){return 0;} void log_plan(const Plan&, double, bool){} Plan::~Plan(){ delete narrow; } }
int main(int argc, char** argv) {
    FILE* f = fopen("probs.txt", "r");
    std::vector<std::vector<long long>> P; int r, e;
    while (fscanf(f, "%d %d", &r, &e) == 2) { std::vector<long long> v{r, e}; for (int i = 0; i < 2 * r; ++i) { long long x; if (fscanf(f, "%lld", &x) != 1) return 1; v.push_back(x); } P.push_back(v); }
    FILE* dump = fopen(argv[1], "w");
    std::vector<tt_plan_options_t> os;
    auto add = [&](auto fn) { tt_plan_options_t o{}; fn(o); os.push_back(o); };
    add([](tt_plan_options_t& o) { o.slot_dims = 1; o.stages = 4; });
    add([](tt_plan_options_t& o) { o.slot_dims = 1; o.stages = 3; });
    add([](tt_plan_options_t& o) { o.sd_vmax = 8192; });
    add([](tt_plan_options_t& o) { o.run_in = 64; });
    add([](tt_plan_options_t& o) { o.run_out = 256; });
    add([](tt_plan_options_t& o) { o.run_in = 32; o.run_out = 512; });
    add([](tt_plan_options_t& o) { o.vector_gather = 1; });
    add([](tt_plan_options_t& o) { o.threads = 256; });
    add([](tt_plan_options_t& o) { o.slots = 4; });
    add([](tt_plan_options_t& o) { o.accumulate = 1; });
    add([](tt_plan_options_t& o) { o.slot_dims = -1; });
    add([](tt_plan_options_t& o) { o.kernel = TT_KERNEL_TILE; });
    add([](tt_plan_options_t& o) { o.stages = 3; });
    DeviceInfo dev;
    for (auto& v : P) {
        int rank = v[0], es = v[1]; int64_t dims[32]; int perm[32];
        for (int i = 0; i < rank; ++i) { dims[i] = v[2 + i]; perm[i] = v[2 + rank + i]; }
        for (auto& o : os) {
            Plan p; p.rank = rank; p.dims.assign(dims, dims + rank); p.perm.assign(perm, perm + rank);
            p.prob = normalize(rank, dims, perm, es, true);
            tt_status_t st = choose_plan(p, dev, &o, nullptr);
            fprintf(dump, "%d %s\n", (int)st, st == TT_SUCCESS ? describe_json(p).c_str() : "");
        }
    }
}
