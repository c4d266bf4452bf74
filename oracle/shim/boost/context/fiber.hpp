// TEST INFRASTRUCTURE ONLY -- not product code, never shipped with libtw_hpccg.
//
// Minimal ucontext stand-in for the slice of boost::context::fiber that the
// reference's Fiber wrapper uses (proj/include/taskweave/fiber.hpp:17-47), so
// the reference's own task-based CPU path (cg_tasks on real threads) can be
// built from its sources for the CPU baseline.
// Boost.Context is not in this image.
//
// Semantics kept: a fiber is a one-shot continuation; std::move(f).resume()
// switches into f and returns the continuation of whoever switched back; the
// entry function receives the caller's continuation and returns the one to
// switch to when it finishes.
#pragma once

#include <ucontext.h>

#include <cstdint>
#include <cstdlib>
#include <functional>
#include <memory>
#include <stdexcept>
#include <utility>

#include "boost/context/fixedsize_stack.hpp"

namespace boost::context {

class fiber;

namespace shim_detail {

struct Ctx {
    ucontext_t uc{};
    char* stack = nullptr;        // owned when this context runs on its own stack
    std::size_t stack_bytes = 0;
    std::function<fiber(fiber&&)> entry;
    Ctx* from = nullptr;          // set by whoever switches into this context
    bool started = false;
    bool finished = false;
    ~Ctx() { std::free(stack); }
};

} // namespace shim_detail

class fiber {
public:
    fiber() noexcept = default;

    template <typename StackAlloc, typename Fn>
    fiber(std::allocator_arg_t, StackAlloc salloc, Fn&& fn) {
        auto* c = new shim_detail::Ctx;
        c->stack_bytes = salloc.size();
        c->stack = static_cast<char*>(std::malloc(c->stack_bytes));
        if (!c->stack) {
            delete c;
            throw std::bad_alloc();
        }
        c->entry = std::forward<Fn>(fn);
        getcontext(&c->uc);
        c->uc.uc_stack.ss_sp = c->stack;
        c->uc.uc_stack.ss_size = c->stack_bytes;
        c->uc.uc_link = nullptr;
        auto bits = reinterpret_cast<std::uintptr_t>(c);
        makecontext(&c->uc, reinterpret_cast<void (*)()>(&fiber::trampoline), 2,
                    static_cast<unsigned>(bits & 0xffffffffu),
                    static_cast<unsigned>(bits >> 32));
        ctx_ = c;
    }

    fiber(fiber&& o) noexcept : ctx_(std::exchange(o.ctx_, nullptr)) {}
    fiber& operator=(fiber&& o) noexcept {
        if (this != &o) {
            reset();
            ctx_ = std::exchange(o.ctx_, nullptr);
        }
        return *this;
    }
    fiber(const fiber&) = delete;
    fiber& operator=(const fiber&) = delete;
    ~fiber() { reset(); }

    explicit operator bool() const noexcept { return ctx_ != nullptr; }
    bool operator!() const noexcept { return ctx_ == nullptr; }

    fiber resume() && {
        shim_detail::Ctx* target = std::exchange(ctx_, nullptr);
        if (!target)
            throw std::logic_error("resume of an empty fiber");
        // The current context becomes a stackless record the target can
        // switch back into.
        auto* self = new shim_detail::Ctx;
        target->from = self;
        target->started = true;
        swapcontext(&self->uc, &target->uc);
        return arrive(self);
    }

private:
    explicit fiber(shim_detail::Ctx* c) noexcept : ctx_(c) {}

    // Runs in the context that was just switched back into.
    static fiber arrive(shim_detail::Ctx* self) {
        shim_detail::Ctx* from = self->from;
        delete self;
        if (from->finished) {
            delete from; // its stack is no longer in use
            return fiber();
        }
        return fiber(from);
    }

    static void trampoline(unsigned lo, unsigned hi) {
        auto* me = reinterpret_cast<shim_detail::Ctx*>(
            (static_cast<std::uintptr_t>(hi) << 32) | static_cast<std::uintptr_t>(lo));
        shim_detail::Ctx* caller = me->from;
        me->from = nullptr;
        shim_detail::Ctx* next = nullptr;
        {
            fiber ret = me->entry(fiber(caller));
            next = std::exchange(ret.ctx_, nullptr);
        }
        if (!next)
            std::abort();
        me->finished = true;
        next->from = me;
        setcontext(&next->uc);
        std::abort();
    }

    void reset() noexcept {
        // A fiber object only ever holds an unstarted context (which owns its
        // stack) or the stackless record of a parked context; dropping the
        // latter abandons it (the reference drops fibers only once done).
        delete ctx_;
        ctx_ = nullptr;
    }

    shim_detail::Ctx* ctx_ = nullptr;
};

} // namespace boost::context
