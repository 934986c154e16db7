// Minimal stand-in for boost::context::fiber (Boost is not installed in this
// image; the reference needs Boost >= 1.70 'context', proj/CMakeLists.txt:13).
//
// ORACLE BUILD SUPPORT ONLY: used to compile the reference VM from
// /root/reference into oracle/_ref/ so it can serve as the CPU checker and the
// CPU baseline.  Implements exactly the surface proj/src/fiber.hpp and
// proj/src/machine.cpp:169-170,304-316,830-833 use:
//   stack_context{size, sp}; fiber(std::allocator_arg, StackAlloc, Fn) where
//   Fn: fiber(fiber&& caller); fiber resume() &&; move; explicit operator bool.
// x86-64 System V only.  A suspended fiber that is destroyed has its stack
// released without unwinding (the VM only does this on an aborted launch).
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <memory>
#include <utility>

extern "C" void forge_shim_ctx_swap(void** save_sp, void* new_sp);

namespace boost {
namespace context {

struct stack_context {
  std::size_t size = 0;
  void* sp = nullptr;
};

class fiber;

namespace shim {

struct record {
  void* sp = nullptr;  // saved stack pointer while suspended
  bool is_thread = false;
  bool finished = false;
  stack_context sctx{};
  std::function<void(stack_context&)> release;
  std::function<fiber(fiber&&)> entry;
};

struct tls_state {
  record thread_rec;       // the OS thread's own context
  record* current = nullptr;
  record* from = nullptr;  // context that just switched away
  tls_state() { thread_rec.is_thread = true; }
};

inline tls_state& tls() {
  static thread_local tls_state s;
  return s;
}

inline void destroy_record(record* r) {
  if (!r || r->is_thread) return;
  auto rel = std::move(r->release);
  stack_context sc = r->sctx;
  delete r;
  if (rel) rel(sc);
}

}  // namespace shim

class fiber {
 public:
  fiber() noexcept = default;

  template <class StackAlloc, class Fn>
  fiber(std::allocator_arg_t, StackAlloc salloc, Fn&& fn) {
    auto* r = new shim::record;
    r->sctx = salloc.allocate();
    r->release = [salloc](stack_context& sc) mutable { salloc.deallocate(sc); };
    r->entry = std::function<fiber(fiber&&)>(std::forward<Fn>(fn));
    // Prime the stack so that the first swap "returns" into trampoline with
    // the SysV call alignment (rsp = 8 mod 16 at function entry).
    auto top = reinterpret_cast<std::uintptr_t>(r->sctx.sp) & ~std::uintptr_t(15);
    auto* slot = reinterpret_cast<void**>(top - 16);
    *slot = reinterpret_cast<void*>(&trampoline);
    void** regs = slot - 6;  // r15 r14 r13 r12 rbx rbp
    for (int i = 0; i < 6; ++i) regs[i] = nullptr;
    r->sp = regs;
    rec_ = r;
  }

  fiber(fiber&& o) noexcept : rec_(std::exchange(o.rec_, nullptr)) {}
  fiber& operator=(fiber&& o) noexcept {
    if (this != &o) {
      reset();
      rec_ = std::exchange(o.rec_, nullptr);
    }
    return *this;
  }
  fiber(const fiber&) = delete;
  fiber& operator=(const fiber&) = delete;
  ~fiber() { reset(); }

  explicit operator bool() const noexcept { return rec_ != nullptr; }

  fiber resume() && {
    shim::record* target = std::exchange(rec_, nullptr);
    auto& t = shim::tls();
    shim::record* self = t.current ? t.current : &t.thread_rec;
    t.from = self;
    t.current = target;
    forge_shim_ctx_swap(&self->sp, target->sp);
    return take_from();
  }

 private:
  explicit fiber(shim::record* r) noexcept : rec_(r) {}

  void reset() noexcept {
    if (rec_ && !rec_->is_thread) shim::destroy_record(rec_);
    rec_ = nullptr;
  }

  // Called right after control arrives in a context: wraps the context that
  // switched to us, or releases it if it has terminated.
  static fiber take_from() {
    auto& t = shim::tls();
    shim::record* f = std::exchange(t.from, nullptr);
    if (!f) return fiber();
    if (f->finished) {
      shim::destroy_record(f);
      return fiber();
    }
    return fiber(f);
  }

  [[noreturn]] static void trampoline() {
    auto& t = shim::tls();
    shim::record* self = t.current;
    fiber next;
    {
      fiber caller = take_from();
      next = self->entry(std::move(caller));
    }
    self->finished = true;
    shim::record* target = std::exchange(next.rec_, nullptr);
    auto& t2 = shim::tls();
    t2.from = self;
    t2.current = target;
    void* dead_sp = nullptr;
    forge_shim_ctx_swap(&dead_sp, target->sp);
    __builtin_unreachable();
  }

  shim::record* rec_ = nullptr;
};

}  // namespace context
}  // namespace boost
