#include "tt_internal.h"
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
namespace tt { int log_level(){return 0;} void log_plan(const Plan&, double, bool){} Plan::~Plan(){ delete narrow; }
namespace model { extern double kBwBytesPerUs, kClockMHz, kIssuePerClk, kTileInstr, kSlotInstr, kSlotInstrSd, kLaunchUs, kRunBytes, kInflightBytes, kTileLatUs, kReadW, kRestW; } }
using namespace tt;
// usage: fit rows.txt key=val ...   rows: rank esize dims.. perm.. run_in run_out
int main(int argc, char** argv) {
    for (int a = 2; a < argc; ++a) {
        char k[64]; double v;
        if (sscanf(argv[a], "%63[^=]=%lf", k, &v) != 2) continue;
        std::string K(k);
        if (K == "slot") model::kSlotInstr = v; else if (K == "slotsd") model::kSlotInstrSd = v;
        else if (K == "tile") model::kTileInstr = v; else if (K == "run") model::kRunBytes = v;
        else if (K == "inflight") model::kInflightBytes = v; else if (K == "lat") model::kTileLatUs = v;
        else if (K == "readw") model::kReadW = v; else if (K == "restw") model::kRestW = v;
        else if (K == "bw") model::kBwBytesPerUs = v; else if (K == "clock") model::kClockMHz = v;
        else if (K == "launch") model::kLaunchUs = v;
    }
    FILE* f = fopen(argv[1], "r");
    int r, e; DeviceInfo dev;
    while (fscanf(f, "%d %d", &r, &e) == 2) {
        int64_t dims[32]; int perm[32]; long long x; int ri, ro;
        for (int i = 0; i < r; ++i) { if (fscanf(f, "%lld", &x) != 1) return 1; dims[i] = x; }
        for (int i = 0; i < r; ++i) { if (fscanf(f, "%d", &perm[i]) != 1) return 1; }
        if (fscanf(f, "%d %d", &ri, &ro) != 2) return 1;
        Plan p; p.rank = r; p.dims.assign(dims, dims + r); p.perm.assign(perm, perm + r);
        p.prob = normalize(r, dims, perm, e, true);
        tt_plan_options_t o{}; o.run_in = ri; o.run_out = ro;
        tt_status_t st;
        if (ri == 0 && ro == 0) {
            int k = widen_factor(p.prob);
            if (k > 1) p.prob = widen_problem(p.prob, k);
            st = choose_plan(p, dev, nullptr, nullptr);
        } else {
            st = choose_plan(p, dev, &o, nullptr);
        }
        if (st != TT_SUCCESS) { printf("nan -\n"); continue; }
        std::string ext = "[";
        for (int i = 0; i < p.tile.a; ++i) ext += (i ? "," : "") + std::to_string(p.tile.tExt[i]);
        ext += "]";
        printf("%.6f %s %d %d\n", p.kc.predicted_us, ext.c_str(), p.kc.kernel, p.kc.sdq ? 1 : 0);
    }
}
