/* forge_shim_ctx_swap(void** save_sp, void* new_sp) — x86-64 SysV context swap
 * for the Boost.Context stand-in (oracle build support only). Saves the
 * callee-saved registers on the current stack, stores rsp to *save_sp, switches
 * to new_sp and restores the registers saved there. */
    .text
    .globl forge_shim_ctx_swap
    .type forge_shim_ctx_swap, @function
forge_shim_ctx_swap:
    pushq %rbp
    pushq %rbx
    pushq %r12
    pushq %r13
    pushq %r14
    pushq %r15
    movq %rsp, (%rdi)
    movq %rsi, %rsp
    popq %r15
    popq %r14
    popq %r13
    popq %r12
    popq %rbx
    popq %rbp
    ret
    .size forge_shim_ctx_swap, .-forge_shim_ctx_swap
    .section .note.GNU-stack,"",@progbits
