// dist.cu -- sharded multi-GPU permutation (placeholder until the NCCL path lands).
#include "tt_internal.h"

extern "C" {

tt_status_t tt_comm_unique_id(void* id) { (void)id; return TT_UNSUPPORTED; }
tt_status_t tt_comm_init(tt_comm_t* comm, const void* id, int nranks, int rank) {
    (void)comm; (void)id; (void)nranks; (void)rank;
    return TT_UNSUPPORTED;
}
tt_status_t tt_comm_destroy(tt_comm_t comm) { (void)comm; return TT_UNSUPPORTED; }
tt_status_t tt_plan_sharded(tt_plan_t* plan, tt_comm_t comm, int rank, const int64_t* global_dims,
                            const int* perm, size_t elem_size, tt_stream_t stream) {
    (void)plan; (void)comm; (void)rank; (void)global_dims; (void)perm; (void)elem_size; (void)stream;
    return TT_UNSUPPORTED;
}
tt_status_t tt_execute_sharded(tt_plan_t plan, const void* in_local, void* out_local) {
    (void)plan; (void)in_local; (void)out_local;
    return TT_UNSUPPORTED;
}
tt_status_t tt_plan_shard_dims(tt_plan_t plan, int64_t* a, int64_t* b) {
    (void)plan; (void)a; (void)b;
    return TT_UNSUPPORTED;
}

}
