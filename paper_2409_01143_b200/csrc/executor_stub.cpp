#include "executor.hpp"
namespace hexexec {
class Executor {};
Executor* make_executor(const std::string&, const std::string&, const std::string&, const std::string&, int, int, int, const void*, size_t) { throw InvalidArgument("executor not built"); }
void executor_step(Executor&, const int32_t*, size_t, float*) {}
void executor_step_async(Executor&) {}
void executor_sync(Executor&) {}
float executor_last_loss(Executor&) { return 0; }
void executor_synth_tokens(const Executor&, int64_t, int32_t*, size_t) {}
bool executor_tensor_info(const Executor&, const std::string&, int64_t*, int64_t*, int64_t*, int64_t*) { return false; }
void executor_read_tensor(Executor&, const std::string&, int, float*, size_t) {}
std::string executor_stats_json(const Executor&) { return "{}"; }
void destroy_executor(Executor* e) { delete e; }
}
